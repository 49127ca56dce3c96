#!/bin/bash
# ncu --set full of the key-side router kernels of one cfg2 forward (router_rows, kprep, project)
ncu --set full --import-source on --clock-control none -k regex:"router_rows|kprep|project_kernel" -c 4 \
    -o gpurun_out/ncu_router -f python bench.py --config cfg2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/ncu_router.log 2>&1
ls -la gpurun_out/ncu_router.ncu-rep
