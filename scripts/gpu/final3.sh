# round-2 closing evidence: bench lines, per-config verification, traffic, launch lists,
# ncu summaries of the kernels changed since the r02 captures
mkdir -p gpurun_out /tmp/reps
python bench.py > gpurun_out/bench_line.txt 2> gpurun_out/bench_err.txt
python bench.py --impl reference > gpurun_out/bench_ref_line.txt 2>> gpurun_out/bench_err.txt
python bench.py --workload batch > gpurun_out/bench_batch_line.txt 2>> gpurun_out/bench_err.txt
python scripts/verify_configs.py > gpurun_out/vc.txt 2>&1
python scripts/traffic_capture.py 8192 > gpurun_out/traffic.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_8192_r02c.csv python scripts/prof_one.py 8192 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_1024_ts32_r02c.csv python scripts/prof_one.py 1024 fp32 32 > /dev/null 2>&1
for spec in "k_chase2:0:8192:fp32:0" "k_chase2:0:1024:fp32:32"; do
IFS=: read k s n dt ts <<< "$spec"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -s $s -c 1 -f -o /tmp/reps/f_${k}_${n} python scripts/prof_one.py $n $dt $ts > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/reps/f_${k}_${n}.ncu-rep > gpurun_out/sum_${k}_${n}.txt
done
tail -c 300 gpurun_out/bench_line.txt; tail -c 300 gpurun_out/bench_ref_line.txt; tail -c 300 gpurun_out/bench_batch_line.txt; tail -3 gpurun_out/vc.txt
