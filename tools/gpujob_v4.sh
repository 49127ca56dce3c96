#!/bin/bash
# v4 sparse kernel: watchdog-build parity check, stage timings vs the product library, trace (analysis helper)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SLA2_LIB=paper_2602_12675_b200/libsla2_v4wd.so timeout 240 python tools/v2_check.py > gpurun_out/v4_check.log 2>&1; rc=$?
echo "v4_check rc=$rc"; tail -12 gpurun_out/v4_check.log
if [ $rc -ne 0 ]; then exit 1; fi
for lib in v4 b200; do
  echo "== $lib"; SLA2_LIB=paper_2602_12675_b200/libsla2_$lib.so timeout 120 python -u tools/fa_prof.py 2>&1 | head -3
done
SLA2_LIB=paper_2602_12675_b200/libsla2_v4tr.so timeout 120 python tools/trace_v4.py > gpurun_out/trace_v4b.txt 2>&1; tail -30 gpurun_out/trace_v4b.txt
