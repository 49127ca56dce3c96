#!/bin/bash
# round-end measurement: default bench line (cfg2), cfg3 / cfg4, reference arm, launch list (analysis helper)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/smi.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "cfg2 rc=$?"
timeout 600 python bench.py --config cfg3 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo "cfg3 rc=$?"
timeout 900 python bench.py --config cfg4 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "cfg4 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-dense > /dev/null 2>&1; echo "ncu rc=$?"
for f in cfg2 cfg3 cfg4 ref; do echo "== $f"; tail -c 1500 gpurun_out/bench_$f.json; tail -3 gpurun_out/bench_$f.err; done
