mkdir -p gpurun_out
show() { python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('ms/step', round(d['ms_per_step'],2), {k: round(v.get('ms') or 0, 2) for k, v in d['phase_roofline'].items()})
"; }
for c in 3 2 1; do echo "cta/sm $c"; BSVD_CTA_PER_SM=$c python bench.py --workload batch --steps 3 --warmup 3 --no-e2e --no-cpu | show; done
