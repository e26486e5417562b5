# C5 stage 3: launch list + ncu of k_slice and k_values_u on the 4096 x 512^2 batch
mkdir -p gpurun_out /tmp/reps
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c5.csv python scripts/prof_batch.py 4096 > /dev/null 2>&1
for k in k_slice k_values_u k_chase_cta; do
timeout 900 ncu --set full --clock-control none -k regex:$k -c 1 -f -o /tmp/reps/c5_$k python scripts/prof_batch.py 4096 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/reps/c5_$k.ncu-rep > gpurun_out/sum_c5_$k.txt
done
head -30 gpurun_out/sum_c5_k_values_u.txt; head -30 gpurun_out/sum_c5_k_slice.txt
