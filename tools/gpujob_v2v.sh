#!/bin/bash
# v2 variants: watchdog-build parity checks, then interleaved forward timings (analysis helper)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in ${CHECKS:-wd}; do
  SLA2_LIB=paper_2602_12675_b200/libsla2_$c.so timeout 240 python tools/v2_check.py > gpurun_out/v2_check_$c.log 2>&1; rc=$?
  echo "check $c rc=$rc"; tail -2 gpurun_out/v2_check_$c.log
  if [ $rc -ne 0 ]; then exit 1; fi
done
for rep in 1 2 3; do for lib in ${LIBS:-b200}; do
  printf "%-8s " $lib; SLA2_LIB=paper_2602_12675_b200/libsla2_$lib.so timeout 120 python -u tools/fa_prof.py 2>&1 | head -1
done; done
