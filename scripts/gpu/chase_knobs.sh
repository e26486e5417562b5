# chase: poll back-off and cluster count
show() { python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('ms/step', round(d['ms_per_step'],2), {k: round(v.get('ms') or 0, 2) for k, v in d['phase_roofline'].items()})
"; }
echo base; python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu | show
for s in 1000000 8 0; do echo "NSPIN=$s"; BSVD_CHASE_NSPIN=$s python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu | show; done
for c in 24 30 37; do echo "CLUSTERS=$c"; BSVD_CHASE_CLUSTERS=$c python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu | show; done
