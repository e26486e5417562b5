for m in 2 3; do echo "TC mode $m"; BSVD_FLAT_TC=$m python scripts/flat_check.py 2>&1 | grep "n=256\|n=2048\|n=3000\|n=8192\|8192 err"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_8192_tc.csv python scripts/prof_one.py 8192 > /dev/null 2>&1
mkdir -p /tmp/reps
for spec in "k_tgemm<1:20" "k_tgemm<2:20"; do
k=${spec%%:*}; s=${spec##*:}; nm=$(echo $k | tr -d '<')
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$k" -s $s -c 1 -f -o /tmp/reps/full_$nm python scripts/prof_one.py 8192 > /dev/null 2>&1
python scripts/ncu_lines.py /tmp/reps/full_$nm.ncu-rep 40 > gpurun_out/lines_$nm.txt
python scripts/ncu_summary.py /tmp/reps/full_$nm.ncu-rep > gpurun_out/sum_$nm.txt
done
