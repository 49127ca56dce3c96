#!/bin/bash
# v2 epilogue variants: parity check, interleaved stage timings, trace (analysis helper)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SLA2_LIB=paper_2602_12675_b200/libsla2_${CHECK:-b200}.so timeout 240 python tools/v2_check.py > gpurun_out/v2_check.log 2>&1; rc=$?
echo "v2_check rc=$rc"; tail -8 gpurun_out/v2_check.log
if [ $rc -ne 0 ]; then exit 1; fi
for rep in 1 2; do for lib in ${LIBS:-v2old b200 v2c32}; do
  echo "== $lib"; SLA2_LIB=paper_2602_12675_b200/libsla2_$lib.so timeout 120 python -u tools/fa_prof.py 2>&1 | head -2
done; done
[ -n "$TRACE" ] && SLA2_LIB=paper_2602_12675_b200/libsla2_b200_trace.so timeout 120 python tools/trace_v2.py > gpurun_out/trace_v2c.txt 2>&1; [ -n "$TRACE" ] && tail -32 gpurun_out/trace_v2c.txt; true
