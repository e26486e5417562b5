"""Stage-3 pass counts on bench.py's input (development aid): the slowest values, traced."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2508_06339_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
gen = torch.Generator(device="cuda")
gen.manual_seed(1000)
x = torch.randn((n, n), generator=gen, device="cuda", dtype=torch.float32)
os.environ["BSVD_S3_STATS"] = "/tmp/w.bin"
v = P.svdvals(x).double().cpu().numpy()
del os.environ["BSVD_S3_STATS"]
st = np.fromfile("/tmp/w.bin", dtype=np.int32).reshape(-1, 8)
tot = st[:, :4].sum(1)
slow = np.argsort(-tot)[:8]
for i in slow:
    nb = [f"{(v[j] - v[i]) / v[0]:.2e}" for j in range(max(0, i - 2), min(n, i + 3)) if j != i]
    print(i, int(tot[i]), st[i][[0, 1, 6, 7]].tolist(), f"sigma {v[i]:.6e}", "gaps/smax", nb, flush=True)
if len(sys.argv) > 2:
    os.environ["BSVD_S3_TRACE"] = str(int(slow[0]))
    P.svdvals(x)
    torch.cuda.synchronize()
