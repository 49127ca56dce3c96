#!/bin/bash
# ncu --set full (source-level) of the persistent sparse kernel in one cfg2 forward -> gpurun_out/ncu_v2.ncu-rep
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:"${K:-sla2_sparse_v3}" -c 1 -f \
    -o gpurun_out/ncu_${TAG:-v2} python bench.py --config ${CFG:-cfg2} --steps 1 --warmup 1 --no-cpu-baseline \
    --no-e2e --no-dense --no-parity > gpurun_out/ncu_${TAG:-v2}.log 2>&1
tail -3 gpurun_out/ncu_${TAG:-v2}.log
