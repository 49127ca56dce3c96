#!/bin/bash
# FP8 P/V mode: watchdog build first (a hang traps instead of spinning), then the product build,
# the cfg3fp8 bench line and cfg2 (no regression on the bf16 kernel)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: # watchdog step done (r02 first FP8 run)

timeout 600 python -m pytest tests/test_gpu_fp8.py -q -s > gpurun_out/fp8_tests.log 2>&1; echo "tests rc=$?"
grep -E "fp8 max|passed|failed|Error" gpurun_out/fp8_tests.log | tail -30
timeout 300 python bench.py --config cfg3fp8 --no-cpu-baseline > gpurun_out/bench_cfg3fp8.json 2> gpurun_out/bench_cfg3fp8.err; echo "cfg3fp8 rc=$?"
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "cfg2 rc=$?"
for f in cfg3fp8 cfg2; do echo "== $f"; python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(f"gpurun_out/bench_{sys.argv[1]}.json").read().strip().splitlines()[-1])
    print({k:d.get(k) for k in ("ms_per_step","value")}, d.get("stages_ms"), d.get("timeline_ms"), d.get("parity",{}).get("max_rel_err_sampled_heads"), d.get("parity",{}).get("mask_rows_mismatched"), d.get("clocks"))
except Exception as e: print("ERR", e)
PY
tail -3 gpurun_out/bench_$f.err; done
