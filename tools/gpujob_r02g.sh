#!/bin/bash
# round-2 closing job: full GPU suite, bench lines (cfg2, cfg3, cfg3fp8, cfg4, reference arm),
# ncu --set full of the FP8 sparse kernel, launch list of cfg3fp8
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/gputests.log 2>&1; echo "tests rc=$?" | tee -a gpurun_out/gputests.log
tail -3 gpurun_out/gputests.log
timeout 600 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "cfg2 rc=$?"
timeout 600 python bench.py --config cfg3 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo "cfg3 rc=$?"
timeout 600 python bench.py --config cfg3fp8 > gpurun_out/bench_cfg3fp8.json 2> gpurun_out/bench_cfg3fp8.err; echo "cfg3fp8 rc=$?"
timeout 900 python bench.py --config cfg4 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "cfg4 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"sla2_sparse_v2_kernel" -c 1 \
    -o gpurun_out/ncu_sparse_v2_f8 -f python bench.py --config cfg3fp8 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/ncu_f8.log 2>&1; echo "ncu full rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg3fp8.csv \
    python bench.py --config cfg3fp8 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-dense > /dev/null 2>&1; echo "ncu launches rc=$?"
for f in cfg2 cfg3 cfg3fp8 cfg4 ref; do echo "== $f"; tail -c 600 gpurun_out/bench_$f.json; echo; tail -2 gpurun_out/bench_$f.err; done
