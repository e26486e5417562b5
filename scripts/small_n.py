"""Small-n timing (development aid): wall time per svdvals call, phase timers,
library launches per call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_06339_b200 as P
L = P._lib.lib()
for n, ts, dt in [(1024, 32, torch.float32), (1024, 64, torch.float32), (1024, 128, torch.float32),
                  (512, 64, torch.float32), (2048, 32, torch.float32), (256, 32, torch.float32)]:
    a = torch.randn(n, n, device="cuda", dtype=dt)
    cfg = P.KernelConfig(tilesize=ts)
    for _ in range(3):
        P.svdvals(a, cfg)
    torch.cuda.synchronize()
    l0 = L.bsvd_launch_counter()
    reps = 10
    t0 = time.perf_counter()
    for _ in range(reps):
        P.svdvals(a, cfg)
    torch.cuda.synchronize()
    dt_ms = (time.perf_counter() - t0) / reps * 1e3
    launches = (L.bsvd_launch_counter() - l0) / reps
    tm = {k: 0.0 for k in P.PHASE_KEYS}
    P.svdvals(a, cfg, timers=tm)
    print(f"n={n} ts={ts}: {dt_ms:.2f} ms/call, {launches:.0f} launches/call, "
          f"stage1 {tm['panel']*1e3:.2f} chase {tm['bidiagonal']*1e3:.2f} values {tm['diagonal']*1e3:.2f} ms", flush=True)
