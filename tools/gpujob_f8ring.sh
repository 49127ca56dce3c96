#!/bin/bash
# FP8 ring shape: product (2 K pairs, 4 V pair slots) vs 3 K pairs + 3 V pair slots
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=$PWD/paper_2602_12675_b200
SLA2_LIB=$L/libsla2_f8r33wd.so timeout 300 python -m pytest tests/test_gpu_fp8.py -q -x > gpurun_out/f8r33_tests.log 2>&1; echo "r33 tests rc=$?"; tail -1 gpurun_out/f8r33_tests.log
summ() { python - "$1" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(round(d["ms_per_step"],4), d.get("stages_ms",{}).get("sparse_kernel"), d.get("parity",{}).get("pass"), d.get("clocks",{}).get("sm_mhz"))
except Exception as e: print("ERR", e)
PY
}
for rep in 1 2 3; do
for v in b200 f8r33; do
SLA2_LIB=$L/libsla2_$v.so timeout 300 python bench.py --config cfg3fp8 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/b_$v.json 2> gpurun_out/b_$v.err; echo -n "$v: "; summ gpurun_out/b_$v.json
done; done
