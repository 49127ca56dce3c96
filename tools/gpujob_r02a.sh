#!/bin/bash
# Round-2 status run (analysis helper): GPU tests, v2/v3 parity checks, cfg2/cfg4 bench lines
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "gputests rc=$?"; tail -3 gpurun_out/gputests.log
timeout 240 python tools/v2_check.py > gpurun_out/v2_check.log 2>&1; echo "v2_check rc=$?"; tail -9 gpurun_out/v2_check.log
SLA2_LIB=paper_2602_12675_b200/libsla2_v3.so timeout 240 python tools/v2_check.py > gpurun_out/v3_check.log 2>&1; echo "v3_check rc=$?"; tail -9 gpurun_out/v3_check.log
for lib in b200 v3; do
  SLA2_LIB=paper_2602_12675_b200/libsla2_$lib.so timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg2_$lib.json 2> gpurun_out/bench_cfg2_$lib.err; echo "bench $lib rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/bench_cfg2_$lib.json').read().strip().splitlines()[-1]);print('$lib',d['ms_per_step'],d['stages_ms'],d['parity'],d.get('dense_same_build'),d['clocks'])" || tail -5 gpurun_out/bench_cfg2_$lib.err
done
timeout 300 python bench.py --config cfg4 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "bench cfg4 rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench_cfg4.json').read().strip().splitlines()[-1]);print('cfg4',d['ms_per_step'],d['stages_ms'],d.get('dense_same_build'))" || tail -5 gpurun_out/bench_cfg4.err
