# stage-1 panel rows per thread (cluster size) at 8192
show() { python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('ms/step', round(d['ms_per_step'],2), {k: round(v.get('ms') or 0, 2) for k, v in d['phase_roofline'].items()})
"; }
for r in 0 8 2; do echo "RPT=$r"; BSVD_FLAT_RPT=$r python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu | show; done
for r in 0 8; do echo "RPT=$r fp16"; BSVD_FLAT_RPT=$r python bench.py --dtype fp16 --steps 3 --warmup 2 --no-e2e --no-cpu | show; done
