mkdir -p gpurun_out
show() { python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print(d['config'].get('workload'), d['config'].get('ts'), 'ms/step', round(d['ms_per_step'],2), {k: round(v.get('ms') or 0, 2) for k, v in d['phase_roofline'].items()}, d.get('phase_ms'))
"; }
for ts in 64 128 32; do python bench.py --workload batch --ts $ts --steps 3 --warmup 3 --no-e2e --no-cpu | show; done
