#!/bin/bash
# QAT: K~ codes on the side stream; the QAT tests and two cfg3 bench lines
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "qat or quant or cfg3 or codes or scores" > gpurun_out/qat_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/qat_tests.log
for i in 1 2; do
timeout 300 python bench.py --config cfg3 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/b_cfg3.json 2> gpurun_out/b_cfg3.err; echo "cfg3 rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/b_cfg3.json").read().strip().splitlines()[-1])
print(d["ms_per_step"], d.get("stages_ms"), d.get("timeline_ms"), d.get("parity",{}).get("pass"), d.get("clocks",{}).get("sm_mhz"))
PY
done
