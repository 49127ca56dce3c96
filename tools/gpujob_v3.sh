#!/bin/bash
# Persistent sparse kernel v3: watchdog-build parity check, then the default bench line (analysis helper)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SLA2_LIB=paper_2602_12675_b200/libsla2_wd.so timeout 180 python tools/v2_check.py > gpurun_out/v3_check.log 2>&1; rc=$?
echo "v3_check rc=$rc" >> gpurun_out/v3_check.log
tail -14 gpurun_out/v3_check.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench_cfg2.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['stages_ms'],d['parity'],d.get('dense_same_build'))"
