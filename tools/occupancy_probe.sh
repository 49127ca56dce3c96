#!/bin/bash
# Occupancy limits and waves of every kernel of one cfg2 forward (ncu launch metrics only).
ncu --metrics launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,launch__occupancy_limit_warps,launch__occupancy_limit_blocks,launch__waves_per_multiprocessor,launch__shared_mem_config_size,launch__grid_size,gpu__time_duration.sum \
    --clock-control none -c 40 --csv --log-file gpurun_out/occ.csv \
    python bench.py --config cfg2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-dense > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.DictReader(open("gpurun_out/occ.csv")))
seen = collections.OrderedDict()
for r in rows:
    k = r["Kernel Name"][:60]
    seen.setdefault(k, {})[r["Metric Name"]] = r["Metric Value"]
for k, m in seen.items():
    print(k)
    for n in sorted(m): print("   ", n, m[n])
PY
