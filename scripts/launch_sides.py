"""Per-side kernel durations from an ncu launch list of one flat stage-1 run
(development aid): python scripts/launch_sides.py gpurun_out/launch_8192.csv"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
seq = [(r[ki].split('(')[0].split('<')[0].replace('void ', ''), float(r[vi].replace(',', '')) / 1e3)
       for r in rows[hi + 1:] if len(r) > vi]
agg = collections.defaultdict(lambda: [0, 0.0])
for nm, v in seq:
    agg[nm][0] += 1; agg[nm][1] += v
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:40s} {v[0]:6d} {v[1]/1e3:9.2f} ms {v[1]/tot*100:5.1f}%")
sides = []; cur = None
for nm, v in seq:
    if 'k_fpanel' in nm:
        cur = {'panel': v}; sides.append(cur)
    elif cur is not None and nm.startswith('flat::'):
        k = nm.split('::')[1]; cur[k] = cur.get(k, 0) + v
for i in [0, 1, 10, 11, 30, 31, 60, 61, 100, 101, 120, 121, len(sides) - 1]:
    if i < len(sides):
        print(i, {k: round(v, 1) for k, v in sides[i].items()})
