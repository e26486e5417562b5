python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('ms/step', round(d['ms_per_step'],2), {k: round(v.get('ms') or 0, 2) for k, v in d['phase_roofline'].items()})
"
python bench.py --n 4096 --dtype fp64 --steps 3 --warmup 3 --no-e2e --no-cpu | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('fp64 4096 ms/step', round(d['ms_per_step'],2), {k: round(v.get('ms') or 0, 2) for k, v in d['phase_roofline'].items()})
"
BSVD_CHASE_TRACE=/tmp/ct.bin python scripts/s3_time.py 2048 u > /dev/null 2>&1 && python scripts/chase2_trace.py /tmp/ct.bin | tail -3
