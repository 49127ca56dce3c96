#!/bin/bash
# FP8 P/V with one ring slot per key-block pair: watchdog build first, then tests and bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SLA2_LIB=$PWD/paper_2602_12675_b200/libsla2_wd.so timeout 300 python -m pytest tests/test_gpu_fp8.py -x -q -k "vs_reference" > gpurun_out/fp8_wd.log 2>&1; echo "wd rc=$?"; tail -3 gpurun_out/fp8_wd.log
timeout 600 python -m pytest tests/test_gpu_fp8.py -q -s > gpurun_out/fp8_tests.log 2>&1; echo "tests rc=$?"
grep -E "fp8 max|passed|failed|Error" gpurun_out/fp8_tests.log | tail -12
summ() { python - "$1" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(round(d["ms_per_step"],4), d.get("stages_ms",{}).get("sparse_kernel"), d.get("parity",{}).get("max_rel_err_sampled_heads"), d.get("parity",{}).get("pass"), d.get("clocks",{}).get("sm_mhz"))
except Exception as e: print("ERR", e)
PY
}
for rep in 1 2; do
timeout 300 python bench.py --config cfg3fp8 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/b_fp8.json 2> gpurun_out/b_fp8.err; echo "fp8 rc=$?"; summ gpurun_out/b_fp8.json
timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-dense > gpurun_out/b_cfg2.json 2> gpurun_out/b_cfg2.err; echo "cfg2 rc=$?"; summ gpurun_out/b_cfg2.json
done
