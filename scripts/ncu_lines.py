"""Warp-stall samples per CUDA source line from an ncu report (needs -lineinfo).
python scripts/ncu_lines.py rep.ncu-rep [top]  -- development aid."""
import csv, subprocess, sys, collections
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
agg = collections.Counter(); text = {}
fname = ""; col = None
for row in csv.reader(out):
    if len(row) == 2 and row[0] == "File Path":
        fname = row[1].split("/")[-1]; continue
    if row and row[0] == "Line No":
        col = row.index("Warp Stall Sampling (All Samples)"); continue
    if col is None or len(row) <= col: continue
    if row[0]:
        key = (fname, int(row[0])); text[key] = row[1]
        try: agg[key] += float(row[col] or 0)
        except ValueError: pass
tot = sum(agg.values()) or 1
for key, v in agg.most_common(top):
    print(f"{100*v/tot:5.1f}% {key[0]}:{key[1]:<5d} {text[key].strip()[:100]}")
