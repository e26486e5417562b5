mkdir -p /tmp/reps gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tgemm -s 40 -c 1 -f -o /tmp/reps/g40 python scripts/prof_one.py 8192 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tgemm -s 44 -c 1 -f -o /tmp/reps/g44 python scripts/prof_one.py 8192 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/reps/g44.ncu-rep | head -3
python scripts/ncu_lines.py /tmp/reps/g40.ncu-rep 30
echo ---
python scripts/ncu_lines.py /tmp/reps/g44.ncu-rep 20
