mkdir -p gpurun_out /tmp/reps
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c5.csv python scripts/prof_batch.py 4096 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open('gpurun_out/launch_c5.csv')))
hi = next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]; ki = h.index('Kernel Name'); mi = h.index('Metric Value')
tot = collections.defaultdict(lambda: [0,0.0])
for r in rows[hi+1:]:
    if len(r) <= mi: continue
    name = r[ki].split('(')[0].replace('void ','').replace('bsvd::','')
    try: v = float(r[mi].replace(',',''))
    except: continue
    tot[name][0]+=1; tot[name][1]+=v
s = sum(v[1] for v in tot.values())
for k,v in sorted(tot.items(), key=lambda x:-x[1][1])[:16]:
    print(f"{k[:60]:60s} {v[0]:5d} {v[1]/1e6:8.2f} ms {v[1]/s*100:5.1f}%")
print("total", s/1e6)
PY
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fpanel2 -s 4 -c 1 -f -o /tmp/reps/c5p python scripts/prof_batch.py 4096 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/reps/c5p.ncu-rep 2>/dev/null | head -20
