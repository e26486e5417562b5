# batched chase: reduce-scatter of the right-op row sums
show() { python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('ms/step', round(d['ms_per_step'],2), {k: round(v.get('ms') or 0, 2) for k, v in d['phase_roofline'].items()})
"; }
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --workload batch --steps 3 --warmup 2 --no-e2e --no-cpu | show
for c in 4 2; do echo "per_sm=$c"; BSVD_CTA_PER_SM=$c python bench.py --workload batch --steps 3 --warmup 2 --no-e2e --no-cpu | show; done
