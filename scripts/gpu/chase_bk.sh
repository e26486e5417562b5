# narrow-tile cluster chase (BKT = 32 / 64) vs the 128 tile
show() { python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('ms/step', round(d['ms_per_step'],2), {k: round(v.get('ms') or 0, 2) for k, v in d['phase_roofline'].items()})
"; }
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python scripts/small_n.py 2>&1 | tail -6
echo "BK=128 forced"; BSVD_CHASE_BK=128 python scripts/small_n.py 2>&1 | tail -6
python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu | show
echo "8192 ts 32"; python bench.py --ts 32 --steps 2 --warmup 2 --no-e2e --no-cpu | show
echo "8192 ts 64"; python bench.py --ts 64 --steps 2 --warmup 2 --no-e2e --no-cpu | show
