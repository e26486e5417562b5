"""Per-kernel DRAM traffic of one svdvals call (development + evidence script,
run on the GPU box):  python scripts/traffic_capture.py [n] -> gpurun_out/traffic_n<n>.json
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over every launch of
scripts/prof_one.py; stage 1 = every launch that is not stage 2/3 or copy-in."""
import collections, csv, json, os, subprocess, sys
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
os.makedirs("gpurun_out", exist_ok=True)
log = f"gpurun_out/traffic_n{n}.csv"
subprocess.run(["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
                "--clock-control", "none", "--csv", "--log-file", log, sys.executable, "scripts/prof_one.py", str(n)],
               check=True, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
rows = list(csv.reader(open(log)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.defaultdict(dict)
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    per[(int(r[ii]), r[ki])][r[mi]] = float(r[vi].replace(",", ""))
agg = collections.defaultdict(lambda: {"launches": 0, "bytes": 0.0, "ns": 0.0})
for (_, name), m in per.items():
    base = name.split("(")[0].split("<")[0].replace("void ", "").split("::")[-1]
    a = agg[base]
    a["launches"] += 1
    a["bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    a["ns"] += m.get("gpu__time_duration.sum", 0.0)
not_s1 = {"k_chase2", "k_chase", "k_chase_cta", "k_chase_seq", "k_values", "k_values_u", "k_slice", "k_copy_in_pad",
          "k_absmax", "k_unscale_values",
          "k_pack_band", "k_extract_bidiag", "k_bisect_prep", "k_clear_band"}
out = {k: v["bytes"] / v["launches"] for k, v in agg.items()}
out[f"stage1_step_n{n}"] = sum(v["bytes"] for k, v in agg.items() if k not in not_s1 and not k.startswith("at"))
out["_kernels"] = {k: dict(v) for k, v in agg.items()}
out["_note"] = (f"dram__bytes_read.sum + dram__bytes_write.sum per launch (kernel keys) and summed over every "
                f"stage-1 launch of one n={n} FP32 svdvals (stage1_step_n{n}); ncu, serialised, cold caches")
json.dump(out, open(f"gpurun_out/traffic_n{n}.json", "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if not k.startswith("_")}, indent=1))
