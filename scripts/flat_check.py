"""Dev check of the flat stage-1 path: values vs fp64 LAPACK, then timing."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_06339_b200 as P

def err(got, a):
    want = torch.linalg.svdvals(torch.from_numpy(a.astype(np.float64)).cuda()).cpu().numpy()
    return float(np.max(np.abs(np.asarray(got, np.float64) - want)) / want[0])

rng = np.random.default_rng(1)
for dt, n, ts in [(np.float32, 128, 128), (np.float32, 256, 128), (np.float32, 384, 128), (np.float32, 200, 64),
                  (np.float32, 1024, 128), (np.float32, 2048, 128), (np.float32, 1024, 64), (np.float16, 512, 128),
                  (np.float32, 3000, 128)]:
    a = rng.standard_normal((n, n)).astype(dt)
    t0 = time.time()
    got = P.svdvals(a, P.KernelConfig(tilesize=ts))
    print(f"{np.dtype(dt).name} n={n} ts={ts}: err {err(got, a):.2e}  ({time.time()-t0:.2f}s)", flush=True)
# rank-deficient / zero / identity
for name, a in [("zero", np.zeros((256, 256), np.float32)), ("eye", np.eye(256, dtype=np.float32)),
                ("rank1", np.outer(rng.standard_normal(300), rng.standard_normal(300)).astype(np.float32))]:
    got = P.svdvals(a, P.KernelConfig(tilesize=128))
    print(name, "err", err(got, a) if a.any() else float(np.max(np.abs(got))))
# batch vs single
b = rng.standard_normal((8, 512, 512)).astype(np.float32)
gb = P.svdvals_batched(b, P.KernelConfig(tilesize=64))
print("batch err", max(err(gb[i], b[i]) for i in range(8)))
# timing
dev = torch.device("cuda")
for n in [4096, 8192]:
    x = torch.randn((n, n), device=dev, generator=torch.Generator(device=dev).manual_seed(0))
    cfg = P.KernelConfig.for_size(n)
    P.svdvals(x, cfg); torch.cuda.synchronize()
    tm = {k: 0.0 for k in P.PHASE_KEYS}
    P.svdvals(x, cfg, timers=tm)
    t0 = time.time(); reps = 3
    for _ in range(reps): P.svdvals(x, cfg)
    torch.cuda.synchronize()
    print(f"n={n} {(time.time()-t0)/reps*1e3:.1f} ms/step; stage1 {tm['panel']*1e3:.1f} chase {tm['bidiagonal']*1e3:.1f} values {tm['diagonal']*1e3:.1f}", flush=True)
if n == 8192:
    xh = x.cpu().numpy()
    got = P.svdvals(x, cfg).cpu().numpy()
    print("8192 err vs fp64 LAPACK", err(got, xh))
