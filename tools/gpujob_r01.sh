# Round-1 evidence job (analysis only; rerun after each kernel change): bench lines for every config, the reference arm, the
# ncu launch list of one default forward and one --set full capture of the sparse kernel.
python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
python bench.py --config cfg2pad --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg2pad.json 2>&1
python bench.py --config cfg3 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/bench_cfg3.json 2>&1
python bench.py --config cfg4 --no-cpu-baseline --steps 10 > gpurun_out/bench_cfg4.json 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_cfg2.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv \
    python tools/profile_forward.py --config cfg2 --iters 2 > /dev/null 2>&1
ncu --set full --import-source on -k regex:sla2_sparse_bf16 --launch-skip 2 -c 1 -o gpurun_out/ncu_sparse_cfg2 \
    python tools/profile_forward.py --config cfg2 > /dev/null 2>&1
for f in cfg2 cfg2pad cfg3 cfg4; do
  python -c "import json;d=json.loads(open('gpurun_out/bench_$f.json').read().strip().splitlines()[-1]);print('$f',round(d['ms_per_step'],4),round(d['value']),round(d['roofline']['frac'],3),d.get('dense_same_build',{}).get('speedup_sla2_vs_dense'),(d.get('e2e') or {}).get('ms_per_step'))"
done
