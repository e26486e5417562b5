mkdir -p /tmp/reps gpurun_out
for spec in "k_tgemm:40" "k_tgemm:42"; do
k=${spec%%:*}; s=${spec##*:}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -s $s -c 1 -f -o /tmp/reps/g_${k}_$s python scripts/prof_one.py 8192 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/reps/g_${k}_$s.ncu-rep > gpurun_out/g1_${k}_$s.txt
ncu -i /tmp/reps/g_${k}_$s.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; v=rows[2]
d=dict(zip(h,v))
for k in ['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','dram__throughput.avg.pct_of_peak_sustained_elapsed','launch__grid_size']:
    print(k, d.get(k))
" >> gpurun_out/g1_${k}_$s.txt
done
cat gpurun_out/g1_*.txt
