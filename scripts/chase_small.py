"""Narrow-band chase check (development aid): k_chase2 forced for b <= 64
(BSVD_CHASE2_MIN=0) vs the default kernels -- accuracy vs LAPACK + time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_06339_b200 as P
from oracle import oracle as O
rng = np.random.default_rng(3)
for n, b, dt in [(300, 32, np.float32), (1024, 32, np.float32), (1024, 64, np.float32), (257, 16, np.float64),
                 (640, 64, np.float64), (100, 8, np.float32), (2048, 32, np.float32), (77, 4, np.float64)]:
    a = np.triu(rng.standard_normal((n, n)))
    a -= np.triu(a, b + 1)
    a = a.astype(dt)
    want = np.linalg.svd(a.astype(np.float64), compute_uv=False)
    d, e = P.band_to_bidiagonal(a, b)
    got = O.bidiagonal_values(d, e)
    err = np.max(np.abs(got - want)) / want[0]
    t = torch.from_numpy(np.asfortranarray(a).T.copy()).cuda()
    P.band_to_bidiagonal(t, b); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3): P.band_to_bidiagonal(t, b)
    torch.cuda.synchronize()
    print(f"n={n} b={b} {np.dtype(dt).name}: err {err:.2e}  {(time.perf_counter()-t0)/3*1e3:.2f} ms", flush=True)
