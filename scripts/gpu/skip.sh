show() { python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('ms/step', round(d['ms_per_step'],2), {k: round(v.get('ms') or 0, 2) for k, v in d['phase_roofline'].items()})
"; }
python scripts/s3_time.py 8192 u
python scripts/s3_time.py 16384 u
python bench.py --workload batch --steps 3 --warmup 3 --no-e2e --no-cpu | show
python -m pytest tests -m gpu -x -q -k "bidiag or values or config" 2>&1 | tail -2
