N=${N:-8192}
mkdir -p /tmp/reps
for spec in ${SPECS:-k_fpanel:20 k_fpanel:120}; do
k=${spec%%:*}; s=${spec##*:}
timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s $s -c 1 -f -o /tmp/reps/full_${k}_$s python scripts/prof_one.py $N > /dev/null 2>&1
python scripts/ncu_lines.py /tmp/reps/full_${k}_$s.ncu-rep 60 > gpurun_out/lines_${k}_$s.txt
python scripts/ncu_summary.py /tmp/reps/full_${k}_$s.ncu-rep > gpurun_out/sum_${k}_$s.txt
done
