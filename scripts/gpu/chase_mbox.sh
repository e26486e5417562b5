# chase: edge mailbox (tagged 64-bit words) vs edge flags
show() { python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('ms/step', round(d['ms_per_step'],2), {k: round(v.get('ms') or 0, 2) for k, v in d['phase_roofline'].items()})
"; }
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for mb in 1 0; do echo "MBOX=$mb"; BSVD_CHASE_MBOX=$mb python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu | show; done
for mb in 1 0; do echo "MBOX=$mb 16384"; BSVD_CHASE_MBOX=$mb python bench.py --n 16384 --steps 2 --warmup 2 --no-e2e --no-cpu | show; done
python scripts/small_n.py 2>&1 | head -2
