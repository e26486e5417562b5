"""Per-value Sturm pass counts of stage 3 (development aid; BSVD_S3_STATS).

usage: s3_stats.py [n] [K ...]
Prints per phase (isolation, Laguerre, probe, final bisection) the mean and
max passes per value and the mean over warps of the warp-max total passes --
the quantity the latency-bound k_values time follows.
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2508_06339_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a = torch.randn(n, n, device="cuda", generator=torch.Generator(device="cuda").manual_seed(5))
for k in sys.argv[2:] or ["1"]:
    if k == "u":
        os.environ.pop("BSVD_VALUES_K", None)
    else:
        os.environ["BSVD_VALUES_K"] = k
    path = f"/tmp/s3stats_{n}_{k}.bin"
    os.environ["BSVD_S3_STATS"] = path
    P.svdvals(a)
    del os.environ["BSVD_S3_STATS"]
    st = np.fromfile(path, dtype=np.int32).reshape(-1, 8)
    tot = st[:, :4].sum(1)
    nw = len(tot) // 32
    wmax = tot[: nw * 32].reshape(nw, 32).max(1)
    names = ["isolation/quad", "laguerre", "probe", "final", "-", "-", "lag-fail", "lag-ok"]
    parts = "  ".join(f"{nm} {st[:, i].mean():.2f}/{st[:, i].max()}" for i, nm in enumerate(names))
    print(f"K={k} n={n}: {parts}  total mean {tot.mean():.2f} warp-max mean {wmax.mean():.2f} max {wmax.max()} (warps >= max-2: {(wmax >= wmax.max() - 2).sum()})", flush=True)
    if os.environ.get("S3_WORST"):
        w = int(np.argmax(wmax))
        print(f"  slowest warp {w}: per lane (quad, lag, fail, lag_ok):")
        for l in range(32):
            r = st[w * 32 + l]
            print(f"    value {w*32+l}: {r[0]} {r[1]} {r[6]} {r[7]}")
        slow = np.argsort(-tot)[:12]
        print("  slowest values:", [(int(i), int(tot[i]), tuple(int(v) for v in st[i][[0, 1, 6, 7]])) for i in slow])
        vals = P.svdvals(a).double().cpu().numpy()
        for i in slow[:6]:
            lo, hi = max(0, i - 2), min(n, i + 3)
            print(f"   value {i}: sigma {vals[i]:.17g}  neighbours rel gaps",
                  [f"{(vals[j] - vals[i]) / vals[i]:.2e}" for j in range(lo, hi) if j != i])
