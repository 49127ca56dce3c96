#!/bin/bash
# split forward timing + ncu --set full of the attention / linsel kernels (analysis helper)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 120 python tools/fa_prof.py > gpurun_out/fa_prof.txt 2>&1; echo "prof rc=$?"; cat gpurun_out/fa_prof.txt
NCU=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"sla2_attn_kernel|sla2_linsel_kernel" -c 3 -f \
    -o gpurun_out/ncu_fa python tools/fa_prof.py > gpurun_out/ncu_fa.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_fa.log
