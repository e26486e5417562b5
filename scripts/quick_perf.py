"""Quick per-stage timing on the GPU (development aid, not the bench)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_06339_b200 as P

def run(n, dtype, ts=None, reps=2):
    a = torch.randn(n, n, dtype=dtype, device="cuda")
    cfg = P.KernelConfig(tilesize=ts) if ts else None
    P.svdvals(a, cfg)  # warm
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter(); v = P.svdvals(a, cfg); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    tm = {}
    P.svdvals(a, cfg, timers=tm)
    fl = 8 / 3 * n ** 3
    print(f"n={n} {dtype} ts={ts or P.KernelConfig.for_size(n).tilesize}: {best*1e3:.1f} ms  {fl/best/1e12:.2f} TF/s  "
          + " ".join(f"{k}={v*1e3:.1f}ms" for k, v in tm.items()), flush=True)

if __name__ == "__main__":
    sizes = [int(x) for x in sys.argv[1:]] or [1024, 2048, 4096]
    for n in sizes:
        run(n, torch.float32)
    run(1024, torch.float32, 32)
    run(2048, torch.float64)
