run() { env $1 python bench.py --config cfg2 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/b.json 2>&1; python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);t=d['timeline_ms'];print(sys.argv[2], round(d['ms_per_step'],4), {k:round(v,3) for k,v in t.items()})" gpurun_out/b.json "$1"; }
for v in ${EXPS:-"X=0" "X=1"}; do run "$v"; done
