"""One svdvals call for ncu captures (development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2508_06339_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
dt = {"fp32": torch.float32, "fp64": torch.float64, "fp16": torch.float16}[sys.argv[2] if len(sys.argv) > 2 else "fp32"]
ts = int(sys.argv[3]) if len(sys.argv) > 3 else 0
a = torch.randn(n, n, device="cuda", dtype=torch.float32).to(dt)
P.svdvals(a, P.KernelConfig(tilesize=ts) if ts else None)
torch.cuda.synchronize()
