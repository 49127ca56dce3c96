#!/bin/bash
# tree-reduced mu for the linear branch: parity suite + cfg2 / cfg3 / cfg3fp8 / cfg4 bench lines
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputests.log
summ() { python - "$1" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(round(d["ms_per_step"],4), d.get("timeline_ms"), (d.get("parity") or {}).get("max_rel_err_sampled_heads"), (d.get("parity") or {}).get("pass"), d.get("clocks",{}).get("sm_mhz"))
except Exception as e: print("ERR", e)
PY
}
for rep in 1 2; do for c in cfg2 cfg3fp8 cfg3; do
timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --no-dense > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err; echo -n "$c: "; summ gpurun_out/b_$c.json
done; done
timeout 600 python bench.py --config cfg4 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/b_cfg4.json 2> gpurun_out/b_cfg4.err; echo -n "cfg4: "; summ gpurun_out/b_cfg4.json
