#!/bin/bash
# ncu --set full of the router's two heaviest kernels at cfg4 (router_rows, pool_project)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for k in router_rows_kernel pool_project_kernel; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$k" -c 1 \
    -o gpurun_out/ncu_cfg4_$k -f python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-dense --no-parity > gpurun_out/ncu_cfg4_$k.log 2>&1; echo "$k rc=$?"
done
