#!/bin/bash
# re-entry check: full GPU suite, then the default bench line
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests.log
timeout 600 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "cfg2 rc=$?"
tail -25 gpurun_out/gputests.log; tail -c 1200 gpurun_out/bench_cfg2.json; tail -3 gpurun_out/bench_cfg2.err
