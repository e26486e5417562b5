# closing lines after the batched-chase change: tests, bench lines, C5 launch list
show() { python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('ms/step', round(d['ms_per_step'],2), {k: round(v.get('ms') or 0, 2) for k, v in d['phase_roofline'].items()})
"; }
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/bench_line.txt 2> gpurun_out/bench_err.txt
python bench.py --workload batch > gpurun_out/bench_batch_line.txt 2>> gpurun_out/bench_err.txt
python bench.py --impl reference > gpurun_out/bench_ref_line.txt 2>> gpurun_out/bench_err.txt
show < gpurun_out/bench_line.txt; show < gpurun_out/bench_batch_line.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c5.csv python scripts/prof_batch.py 4096 > /dev/null 2>&1
