# stage-3 block size on the batch (C5) workload
show() { python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('ms/step', round(d['ms_per_step'],2), {k: round(v.get('ms') or 0, 2) for k, v in d['phase_roofline'].items()})
"; }
for t in 0 64 256 32; do echo "VB=$t"; BSVD_VALUES_BLOCK=$t python bench.py --workload batch --steps 3 --warmup 2 --no-e2e --no-cpu | show; done
for p in 2 8; do echo "SLICE_PER=$p"; BSVD_SLICE_PER=$p python bench.py --workload batch --steps 3 --warmup 2 --no-e2e --no-cpu | show; done
