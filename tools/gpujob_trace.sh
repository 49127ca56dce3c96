#!/bin/bash
# v2 timeline + one ncu --set full capture of the persistent kernel (analysis helper)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SLA2_LIB=paper_2602_12675_b200/libsla2_b200_trace.so timeout 120 python tools/trace_v3.py > gpurun_out/trace_v3.txt 2>&1
cat gpurun_out/trace_v3.txt
TAG=${TAG:-v3} timeout 400 bash tools/ncu_v2.sh
ls -la gpurun_out/*.ncu-rep

