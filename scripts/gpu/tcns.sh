# stage-1 W-product split count at 8192 / 16384
show() { python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('ms/step', round(d['ms_per_step'],2), {k: round(v.get('ms') or 0, 2) for k, v in d['phase_roofline'].items()})
"; }
for v in "" "BSVD_TC_NS=1" "BSVD_TC_NS=2" "BSVD_TC_NS=3" "BSVD_TC_NS=4" "BSVD_GRAM_JOINT=1" "BSVD_TC_NOPF=1"; do echo "[$v]"; env $v python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu | show; done
