#!/bin/bash
# round-2 last check on HEAD: full GPU suite, smoke, default bench line
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo "tests rc=$?" | tee -a gpurun_out/gputests.log; tail -3 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "cfg2 rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_cfg2.json").read().strip().splitlines()[-1])
print(d["ms_per_step"], d["value"], d["roofline"]["frac"], d["parity"]["pass"], d["dense_same_build"]["speedup_sla2_vs_dense"], d["clocks"], d["gpu_launches"])
PY
