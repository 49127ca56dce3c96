#!/bin/bash
# router_rows_kernel at 4 CTAs / SM (64 registers) vs 3 (80): cfg2 and cfg4 interleaved
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=$PWD/paper_2602_12675_b200
SLA2_LIB=$L/libsla2_rr4.so timeout 600 python -m pytest tests -m gpu -q -x -k "router or cfg4 or tn2048" > gpurun_out/rr4_tests.log 2>&1; echo "rr4 tests rc=$?"; tail -1 gpurun_out/rr4_tests.log
summ() { python - "$1" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(round(d["ms_per_step"],4), d.get("timeline_ms",{}).get("router_back_done"), (d.get("parity") or {}).get("pass"), d.get("clocks",{}).get("sm_mhz"))
except Exception as e: print("ERR", e)
PY
}
for rep in 1 2; do for v in b200 rr4; do for c in cfg2 cfg4; do
SLA2_LIB=$L/libsla2_$v.so timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --no-dense --no-parity > gpurun_out/b_${v}_$c.json 2> gpurun_out/b_${v}_$c.err; echo -n "$v $c: "; summ gpurun_out/b_${v}_$c.json
done; done; done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:router_rows -c 2 python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-dense --no-parity 2>&1 | grep -E "router_rows|gpu__time" | head -4
SLA2_LIB=$L/libsla2_rr4.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:router_rows -c 2 python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-dense --no-parity 2>&1 | grep -E "router_rows|gpu__time" | head -4
