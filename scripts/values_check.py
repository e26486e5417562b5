"""Stage-3 variants (development aid): time + bitwise agreement of the values
across BSVD_VALUES_K settings on the same bidiagonal."""
import os, sys, time, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_06339_b200 as P
rng = np.random.default_rng(11)
res = {}
for n in (1024, 8192):
    a = torch.randn(n, n, device="cuda", generator=torch.Generator(device="cuda").manual_seed(n))
    band = P.banddiag(a, P.KernelConfig.for_size(n))
    d, e = P.band_to_bidiagonal(band, P.KernelConfig.for_size(n).tilesize)
    P.bidiagonal_values(d, e); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3): v = P.bidiagonal_values(d, e)
    torch.cuda.synchronize()
    np.save(f"gpurun_out/vals_{n}_{os.environ.get('BSVD_VALUES_K','def')}.npy", v.cpu().numpy())
    print(f"K={os.environ.get('BSVD_VALUES_K','def')} n={n}: {(time.perf_counter()-t0)/3*1e3:.2f} ms", flush=True)
