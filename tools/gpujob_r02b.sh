#!/bin/bash
# Sparse-kernel analysis (helper): TMEM/MUFU microbenchmarks, v2/v3 timelines, ncu of both kernels
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 120 tools/bin/mb_tmem > gpurun_out/mb_tmem.txt 2>&1; echo "mb_tmem rc=$?"
timeout 120 tools/bin/mb_tma > gpurun_out/mb_tma.txt 2>&1; echo "mb_tma rc=$?"
SLA2_LIB=paper_2602_12675_b200/libsla2_b200_trace.so timeout 120 python tools/trace_v2.py > gpurun_out/trace_v2.txt 2>&1; echo "trace v2 rc=$?"
SLA2_LIB=paper_2602_12675_b200/libsla2_v3tr.so timeout 120 python tools/trace_v3.py > gpurun_out/trace_v3.txt 2>&1; echo "trace v3 rc=$?"
K=sla2_sparse_v2 TAG=v2 timeout 400 bash tools/ncu_v2.sh
SLA2_LIB=paper_2602_12675_b200/libsla2_v3.so K=sla2_sparse_v3 TAG=v3 timeout 400 bash tools/ncu_v2.sh
ls -la gpurun_out/
