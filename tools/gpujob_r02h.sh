#!/bin/bash
# round-2 final: full GPU suite, smoke, bench lines (cfg2 default, cfg3fp8, cfg4fp8), FP8 ncu
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/gputests.log 2>&1; echo "tests rc=$?" | tee -a gpurun_out/gputests.log
tail -3 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "cfg2 rc=$?"
timeout 600 python bench.py --config cfg3fp8 > gpurun_out/bench_cfg3fp8.json 2> gpurun_out/bench_cfg3fp8.err; echo "cfg3fp8 rc=$?"
timeout 900 python bench.py --config cfg4fp8 --no-cpu-baseline > gpurun_out/bench_cfg4fp8.json 2> gpurun_out/bench_cfg4fp8.err; echo "cfg4fp8 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"sla2_sparse_v2_kernel" -c 1 \
    -o gpurun_out/ncu_sparse_v2_f8 -f python bench.py --config cfg3fp8 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-dense --no-parity > gpurun_out/ncu_f8.log 2>&1; echo "ncu full rc=$?"
for f in cfg2 cfg3fp8 cfg4fp8; do echo "== $f"; python - "$f" <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/bench_{sys.argv[1]}.json").read().strip().splitlines()[-1])
r=d.get("roofline",{}); ds=d.get("dense_same_build") or {}
print(round(d["ms_per_step"],4), "sparse", round(r.get("launch_ms",0),4), "frac", round(r.get("frac",0),3), "dense x", ds.get("speedup_sla2_vs_dense"), "sdpa x", d.get("speedup_vs_sdpa"), "parity", (d.get("parity") or {}).get("pass"), d.get("clocks"))
PY
tail -2 gpurun_out/bench_$f.err; done
