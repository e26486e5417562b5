# FP64 (tree stage 1) knob sweep at 8192
show() { python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('ms/step', round(d['ms_per_step'],2), {k: round(v.get('ms') or 0, 2) for k, v in d['phase_roofline'].items()})
"; }
for v in "" "BSVD_LEAF2=0" "BSVD_LEAF_FT_MIN=16" "BSVD_LEAF_FT_MIN=64" "BSVD_PANEL_NOPRIO=1" "BSVD_NO_OVERLAP=1"; do
  echo "[$v]"; env $v python bench.py --dtype fp64 --steps 2 --warmup 1 --no-e2e --no-cpu | show
done
echo "[ts 64]"; python bench.py --dtype fp64 --ts 64 --steps 2 --warmup 1 --no-e2e --no-cpu | show
