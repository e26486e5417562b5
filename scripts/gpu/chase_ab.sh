# chase A/B: parity suite + 8192 / 16384 step phases
mkdir -p gpurun_out
show() { python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('ms/step', round(d['ms_per_step'],2), {k: round(v.get('ms') or 0, 2) for k, v in d['phase_roofline'].items()})
"; }
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu | show
python bench.py --n 16384 --steps 3 --warmup 2 --no-e2e --no-cpu | show
python scripts/small_n.py 2>&1 | tail -6
