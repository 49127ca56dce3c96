#!/bin/bash
# ncu --set full of one kernel (regex $1) of one forward of config $3 -> gpurun_out/ncu_$2.ncu-rep
ncu --set full --import-source on --clock-control none -k regex:"$1" -c 1 \
    -o gpurun_out/ncu_$2 -f python bench.py --config $3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/ncu_$2.log 2>&1
