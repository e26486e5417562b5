"""Top source lines / SASS by warp-stall samples from an ncu report (development aid).
python scripts/ncu_hot.py rep.ncu-rep [n]"""
import csv, subprocess, sys, collections
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
# find header
i = next(k for k, l in enumerate(out) if l.startswith('"Address"') or l.startswith('"Line"') or l.startswith('"#"'))
rows = list(csv.reader(out[i:]))
hdr = rows[0]
print(hdr[:4])
col = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[col] or 0) for r in rows[1:] if len(r) > col)
rs = sorted(rows[1:], key=lambda r: -float(r[col] or 0) if len(r) > col else 0)[:top]
for r in rs:
    print(f"{100*float(r[col])/tot:5.1f}%  {r[0][:12]} {r[1][:110]}")
