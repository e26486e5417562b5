# batched partial-sum loads in k_fgram / k_fw2x1
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python scripts/small_n.py 2>&1 | head -6
show() { python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('ms/step', round(d['ms_per_step'],2), {k: round(v.get('ms') or 0, 2) for k, v in d['phase_roofline'].items()})
"; }
python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu | show
python bench.py --workload batch --steps 3 --warmup 2 --no-e2e --no-cpu | show
