# chase A/B over BSVD_CHASE_AB bits (4: CTA poll, 8: late edge)
show() { python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('ms/step', round(d['ms_per_step'],2), {k: round(v.get('ms') or 0, 2) for k, v in d['phase_roofline'].items()})
"; }
for ab in 0 4 8 12 0 12; do
  echo "AB=$ab"; BSVD_CHASE_AB=$ab python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu | show
done
for ab in 0 12; do
  echo "AB=$ab 16384"; BSVD_CHASE_AB=$ab python bench.py --n 16384 --steps 2 --warmup 2 --no-e2e --no-cpu | show
done
