#!/bin/bash
# sparse_fa check (watchdog build) then timings: split forward stages, dense (analysis helper)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SLA2_LIB=paper_2602_12675_b200/libsla2_fawd.so timeout 150 python tools/fa_check.py > gpurun_out/fa_check.log 2>&1; rc=$?
echo "fa_check rc=$rc"; tail -16 gpurun_out/fa_check.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 120 python -u tools/fa_prof.py 2>&1 | tee gpurun_out/fa_prof.txt; SLA2_LIB=paper_2602_12675_b200/libsla2_fatr.so timeout 120 python tools/trace_fa.py > gpurun_out/trace_fa_sparse.txt 2>&1; tail -4 gpurun_out/trace_fa_sparse.txt
if [ -n "$NCU" ]; then
NCU=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"sla2_attn_kernel|sla2_linsel_kernel" -c 3 -f \
    -o gpurun_out/ncu_fa python tools/fa_prof.py > gpurun_out/ncu_fa.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_fa.log
fi
