#!/bin/bash
# Round-2 final numbers (analysis helper): GPU suite, bench cfg2 (default line), cfg3, cfg4, cfg5 sweep
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "gputests rc=$?"; tail -2 gpurun_out/gputests.log
timeout 400 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "bench cfg2 rc=$?"
for c in cfg3 cfg4; do timeout 400 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"; done
timeout 900 python bench.py --config cfg5 --steps 5 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo "bench cfg5 rc=$?"
