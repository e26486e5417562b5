# stage 1 as a CUDA graph vs direct enqueue
show() { python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('ms/step', round(d['ms_per_step'],2), 'e2e', round((d.get('e2e') or {}).get('ms_per_step') or 0, 2), {k: round(v.get('ms') or 0, 2) for k, v in d['phase_roofline'].items()})
"; }
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python scripts/small_n.py 2>&1 | head -6
echo "[no graph]"; BSVD_NO_GRAPH=1 python scripts/small_n.py 2>&1 | head -6
for v in "" "BSVD_NO_GRAPH=1"; do echo "[$v]"; env $v python bench.py --steps 5 --warmup 3 --no-cpu | show; done
for v in "" "BSVD_NO_GRAPH=1"; do echo "[$v batch]"; env $v python bench.py --workload batch --steps 3 --warmup 2 --no-e2e --no-cpu | show; done
