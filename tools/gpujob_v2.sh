#!/bin/bash
# Persistent sparse kernel check: parity vs v1 / oracle, then the default bench line (analysis helper)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 240 python tools/v2_check.py > gpurun_out/v2_check.log 2>&1; echo "v2_check rc=$?" >> gpurun_out/v2_check.log
tail -12 gpurun_out/v2_check.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_cfg2.json; tail -5 gpurun_out/bench_cfg2.err
