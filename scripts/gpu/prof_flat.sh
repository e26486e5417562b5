N=${N:-8192}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_$N.csv python scripts/prof_one.py $N > /dev/null 2>&1
mkdir -p /tmp/reps
for k in ${KS:-k_fpanel k_fgemm1 k_fgemm2 k_fw2x1 k_fgram}; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s ${SKIP:-20} -c 1 -f -o /tmp/reps/full_$k python scripts/prof_one.py $N > /dev/null 2>&1
ncu -i /tmp/reps/full_$k.ncu-rep --page raw --csv > gpurun_out/raw_$k.csv
ncu -i /tmp/reps/full_$k.ncu-rep --page source --csv > gpurun_out/src_$k.csv 2>/dev/null
python scripts/ncu_summary.py /tmp/reps/full_$k.ncu-rep > gpurun_out/sum_$k.txt
done
ls -la gpurun_out
