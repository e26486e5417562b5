mkdir -p /tmp/reps
for s in 40 41; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tgemm -s $s -c 1 -f -o /tmp/reps/tg_$s python scripts/prof_one.py 8192 > /dev/null 2>&1
python scripts/ncu_lines.py /tmp/reps/tg_$s.ncu-rep 40 > gpurun_out/lines_tg_$s.txt
python scripts/ncu_summary.py /tmp/reps/tg_$s.ncu-rep > gpurun_out/sum_tg_$s.txt
done
