"""Batch (C5) phase timing (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_06339_b200 as P
x = torch.randn(4096, 512, 512, device="cuda")
P.svdvals_batched(x[:64]); torch.cuda.synchronize()
tm = {k: 0.0 for k in P.PHASE_KEYS}
P.svdvals_batched(x, timers=tm); torch.cuda.synchronize()
t0 = time.perf_counter(); P.svdvals_batched(x); torch.cuda.synchronize()
print(f"CTA_PER_SM={os.environ.get('BSVD_CTA_PER_SM','max')}: {(time.perf_counter()-t0)*1e3:.1f} ms; stage1 {tm['panel']*1e3:.1f} chase {tm['bidiagonal']*1e3:.1f} values {tm['diagonal']*1e3:.1f}", flush=True)
