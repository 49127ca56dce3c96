#!/bin/bash
# sparse_fa check (watchdog build) then per-variant timings (analysis helper)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SLA2_LIB=paper_2602_12675_b200/libsla2_fawd.so timeout 150 python tools/fa_check.py > gpurun_out/fa_check.log 2>&1; rc=$?
echo "fa_check rc=$rc"; tail -16 gpurun_out/fa_check.log | grep -v "^B1 H1 N2048"
if [ $rc -ne 0 ]; then exit 1; fi
for lib in ${LIBS:-b200}; do
  echo "== $lib"; SLA2_LIB=paper_2602_12675_b200/libsla2_$lib.so timeout 120 python -u tools/fa_prof.py 2>&1 | tee gpurun_out/fa_prof_$lib.txt
done
