show() { python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('ms/step', round(d['ms_per_step'],2), {k: round(v.get('ms') or 0, 2) for k, v in d['phase_roofline'].items()})
"; }
for r in 0 8 4; do echo "rpt $r"; if [ $r = 0 ]; then python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu | show; else BSVD_FLAT_RPT=$r python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu | show; fi; done
