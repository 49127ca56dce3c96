#!/bin/bash
# GPU suite + bench lines (cfg2 default, cfg3, cfg4) for the current build (analysis helper)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "gputests rc=$?"; tail -3 gpurun_out/gputests.log
timeout 400 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "bench cfg2 rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench_cfg2.json').read().strip().splitlines()[-1]);print('cfg2',d['ms_per_step'],d['stages_ms'],d['parity']['pass'],d.get('dense_same_build'),d.get('torch_sdpa_ms'),d['e2e']['ms_per_step'],d['cpu_baseline']['value'],d['clocks'])" || tail -5 gpurun_out/bench_cfg2.err
for c in cfg3 cfg4; do
timeout 400 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1]);print('$c',d['ms_per_step'],d['stages_ms'],(d['parity'] or {}).get('pass'),d.get('dense_same_build'),d['clocks']['sm_mhz'])" || tail -5 gpurun_out/bench_$c.err
done
