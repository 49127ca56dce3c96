#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python bench.py --config cfg5fp8 > gpurun_out/bench_cfg5fp8.json 2> gpurun_out/bench_cfg5fp8.err; echo "cfg5fp8 rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_cfg5fp8.json").read().strip().splitlines()[-1])
for p in d["sweep"]: print(p["N"], p["sparsity_pct"], round(p["sla2_ms"],3), round(p["speedup_vs_dense"],1), round(p["speedup_vs_sdpa"],1))
PY
tail -2 gpurun_out/bench_cfg5fp8.err
