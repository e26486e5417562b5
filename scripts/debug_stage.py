"""Localise a parity failure by stage (development aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2508_06339_b200 as P
from oracle import oracle as O

def sv(x):
    return np.linalg.svd(np.asarray(x, np.float64), compute_uv=False)

for n, ts, dt in [(256, 64, np.float64), (320, 64, np.float64), (300, 64, np.float64), (192, 64, np.float64),
                  (128, 64, np.float64), (64, 64, np.float64), (300, 32, np.float64), (320, 128, np.float64)]:
    a = np.random.default_rng(n + ts).standard_normal((n, n)).astype(dt)
    ref = sv(a)
    band = P.banddiag(a, P.KernelConfig(tilesize=ts))
    e1 = np.max(np.abs(sv(band)[:n] - ref)) / ref[0]
    # band structure
    npad = band.shape[0]
    off = np.abs(np.triu(band, ts + 1)).max() + np.abs(np.tril(band, -1)).max()
    _, oband, _, _ = O.svdvals(a, ts, return_stages=True)
    d, e = P.band_to_bidiagonal(oband, ts)
    bd = np.diag(d) + np.diag(e, 1)
    e2 = np.max(np.abs(sv(bd)[:n] - ref)) / ref[0]
    v = P.svdvals(a, P.KernelConfig(tilesize=ts))
    e3 = np.max(np.abs(v - ref)) / ref[0]
    print(f"n={n} ts={ts}: stage1(tree) {e1:.2e} offband {off:.1e} | stage2(on oracle band) {e2:.2e} | full {e3:.2e}", flush=True)
