"""Median stage-3 device time over repeated svdvals calls (development aid).

usage: s3_time.py [n] [K ...]   -- K = BSVD_VALUES_K variants to time (default: as set)
Also checks that every variant returns the first variant's values bit for bit.
"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_06339_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
ks = sys.argv[2:] or [os.environ.get("BSVD_VALUES_K", "1")]
a = torch.randn(n, n, device="cuda", generator=torch.Generator(device="cuda").manual_seed(5))
first = None
for k in ks:
    if k == "u":
        os.environ.pop("BSVD_VALUES_K", None)
    else:
        os.environ["BSVD_VALUES_K"] = k
    v = P.svdvals(a)
    ts = []
    for _ in range(7):
        tm = {kk: 0.0 for kk in P.PHASE_KEYS}
        P.svdvals(a, timers=tm)
        ts.append(tm["diagonal"] * 1e3)
    same = "" if first is None else ("  same bits" if torch.equal(v, first) else
                                     f"  DIFFERS max {float((v - first).abs().max() / first[0]):.2e}")
    first = v if first is None else first
    print(f"{os.environ.get('TAG','')} K={k} n={n} stage3 median {statistics.median(ts):.2f} ms "
          f"(min {min(ts):.2f} max {max(ts):.2f}){same}", flush=True)
