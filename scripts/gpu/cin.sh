show() { python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('ms/step', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],3) if d.get('e2e') else None, {k: round(v.get('ms') or 0, 2) for k, v in d['phase_roofline'].items()})
"; }
python bench.py --workload batch --steps 3 --warmup 3 --no-e2e --no-cpu | show
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu | show
python bench.py --n 1024 --ts 32 --steps 10 --warmup 3 --no-e2e --no-cpu | show
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_absmax|k_copy_in_pad" --csv python scripts/prof_batch.py 4096 2>/dev/null | grep -E "k_absmax|k_copy" | cut -c1-40,150-400 | head
