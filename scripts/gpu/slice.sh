show() { python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('ms/step', round(d['ms_per_step'],2), {k: round(v.get('ms') or 0, 2) for k, v in d['phase_roofline'].items()})
"; }
for p in 1 2 4; do echo "slice per $p"; BSVD_SLICE_PER=$p python bench.py --workload batch --steps 3 --warmup 3 --no-e2e --no-cpu | show; done
for p in 1 2; do BSVD_SLICE_PER=$p TAG=slice$p python scripts/s3_time.py 1024 u; done
python scripts/s3_time.py 1024 u
