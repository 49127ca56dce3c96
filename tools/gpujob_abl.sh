#!/bin/bash
# Sparse-kernel ablations (analysis): sparse kernel ms at cfg2 for each variant library
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for lib in ${LIBS:-b200 v2 nohsel noexp both}; do
  SLA2_LIB=paper_2602_12675_b200/libsla2_$lib.so timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-dense --no-parity --steps 20 > gpurun_out/abl_$lib.json 2>gpurun_out/abl_$lib.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/abl_$lib.json').read().strip().splitlines()[-1]);print('$lib',round(d['stages_ms']['sparse_kernel'],4),round(d['ms_per_step'],4),d['clocks']['sm_mhz'])" || tail -3 gpurun_out/abl_$lib.err
done
