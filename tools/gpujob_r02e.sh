#!/bin/bash
# new dense tests + ncu --set full of the round-2 kernels (analysis helper)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k dense 2>&1 | tail -2
NCU=1 timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"sla2_attn_kernel" -c 1 -f -o gpurun_out/ncu_dense_r02 python tools/fa_prof.py > /dev/null 2>&1; echo "ncu dense rc=$?"
NCU=1 H=12 timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"attn_i8|linsel|quant_prep" -c 4 -f -o gpurun_out/ncu_qat_r02 python tools/qat_prof.py > /dev/null 2>&1; echo "ncu qat rc=$?"
