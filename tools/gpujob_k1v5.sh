#!/bin/bash
# sparse_v2 ring shape: 1 K pair + 5 V slots vs the product's 2 + 4 (bf16 and FP8), interleaved
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=$PWD/paper_2602_12675_b200
SLA2_LIB=$L/libsla2_k1v5wd.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp8.py -q -x -k "forward_bf16 or vs_reference or ragged or budget" > gpurun_out/k1_tests.log 2>&1; echo "k1v5 tests rc=$?"; tail -1 gpurun_out/k1_tests.log
summ() { python - "$1" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(round(d["ms_per_step"],4), d.get("stages_ms",{}).get("sparse_kernel"), d.get("clocks",{}).get("sm_mhz"))
except Exception as e: print("ERR", e)
PY
}
for rep in 1 2; do for v in b200 k1v5; do for c in cfg2 cfg3fp8; do
SLA2_LIB=$L/libsla2_$v.so timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --no-dense --no-parity > gpurun_out/b_${v}_$c.json 2> gpurun_out/b_${v}_$c.err; echo -n "$v $c: "; summ gpurun_out/b_${v}_$c.json
done; done; done
