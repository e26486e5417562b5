# fused copy-in + max|a| (relaxed normalisation): parity + step
show() { python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('ms/step', round(d['ms_per_step'],2), 'e2e', round(d.get('e2e',{}).get('ms_per_step') or 0,2), {k: round(v.get('ms') or 0, 2) for k, v in d['phase_roofline'].items()})
"; }
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 --no-cpu | show
python bench.py --workload batch --steps 3 --warmup 2 --no-cpu | show
