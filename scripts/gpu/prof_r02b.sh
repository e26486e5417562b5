N=8192
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_8192_v2.csv python scripts/prof_one.py $N > /dev/null 2>&1
mkdir -p /tmp/reps
for spec in "k_tgemm:40" "k_tgemm:41" "k_tgemm:42" "k_fpanel2:20" "k_fpanel2:120" "k_chase2:0" "k_values_u:0" "k_fw2x1:40" "k_tbuild:40"; do
k=${spec%%:*}; s=${spec##*:}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -s $s -c 1 -f -o /tmp/reps/f_${k}_$s python scripts/prof_one.py $N > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/reps/f_${k}_$s.ncu-rep > gpurun_out/sum_${k}_$s.txt
ncu -i /tmp/reps/f_${k}_$s.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; v=rows[2]
d=dict(zip(h,v))
for k in ['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active','dram__throughput.avg.pct_of_peak_sustained_elapsed','lts__throughput.avg.pct_of_peak_sustained_elapsed','sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum']:
    print(k, d.get(k))
" >> gpurun_out/sum_${k}_$s.txt
done
cuobjdump -sass paper_2508_06339_b200/lib/libbsvd.so 2>/dev/null | grep -o "UTCMMA\|UTCHMMA\|UTMALDG\|UBLKCP\|LDTM\|UTCBAR" | sort | uniq -c > gpurun_out/sass_tc_mnemonics.txt
