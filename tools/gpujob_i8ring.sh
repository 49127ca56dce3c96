#!/bin/bash
# attn_i8 ring depth: product (4) vs 5 vs 6 key/V code slots per lane, cfg3 interleaved
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=$PWD/paper_2602_12675_b200
SLA2_LIB=$L/libsla2_i8r6.so timeout 600 python -m pytest tests -m gpu -q -x -k "qat or cfg3 or codes or scores" > gpurun_out/i8r6_tests.log 2>&1; echo "r6 tests rc=$?"; tail -1 gpurun_out/i8r6_tests.log
summ() { python - "$1" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(round(d["ms_per_step"],4), d.get("stages_ms",{}).get("sparse_kernel"), d.get("parity",{}).get("pass"), d.get("clocks",{}).get("sm_mhz"))
except Exception as e: print("ERR", e)
PY
}
for rep in 1 2; do
for v in b200 i8r5 i8r6; do
SLA2_LIB=$L/libsla2_$v.so timeout 300 python bench.py --config cfg3 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/b_$v.json 2> gpurun_out/b_$v.err; echo -n "$v: "; summ gpurun_out/b_$v.json
done; done
