# which dependency binds the chase: skip block-flag (16) / mailbox (32) waits (timing only)
show() { python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('ms/step', round(d['ms_per_step'],2), {k: round(v.get('ms') or 0, 2) for k, v in d['phase_roofline'].items()})
"; }
for dg in 0 16 32 48; do echo "DIAG=$dg"; BSVD_CHASE_DIAG=$dg python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu 2>&1 | show; done
for dg in 0 48; do echo "DIAG=$dg 16384"; BSVD_CHASE_DIAG=$dg python bench.py --n 16384 --steps 2 --warmup 1 --no-e2e --no-cpu 2>&1 | show; done
