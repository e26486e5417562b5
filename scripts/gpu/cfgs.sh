mkdir -p gpurun_out
show() { python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print(d['config'].get('workload'), d['config'].get('n'), 'ms/step', round(d['ms_per_step'],2))
for k,v in d['phase_roofline'].items(): print('   ', k, {kk: vv for kk, vv in v.items() if kk in ('ms','achieved','frac')})
"; }
python bench.py --workload batch --steps 3 --warmup 3 --no-e2e --no-cpu | show
python bench.py --n 1024 --ts 32 --steps 10 --warmup 3 --no-e2e --no-cpu | show
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu | show
