"""Generate the split-K fixtures tests/golden/splitk_*.npz from the REFERENCE
implementation itself (geqrt_splitk / tsqrt_splitk, kernels.py:233-361,
:459-515, reached through KernelConfig.splitk).  Run in the build container:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python scripts/make_golden_splitk.py

The reference's own tests only pin splitk through its tune grid; these cases
cover even / odd / maximal split counts, ragged segments (ts not divisible by
splitk) and all three precisions, for the GEQRT tile kernel and the whole
stage-1 band (bit-exact targets for the oracle and the faithful GPU path).
"""
from __future__ import annotations

import os
import sys

import numpy as np

import bandsvd as B
from bandsvd import (DenseMatrix, KernelConfig, ParallelBackend, TauStore, banddiag, band_to_bidiagonal,
                     svdvals)
from bandsvd.matrix import pad_to_tiles

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def pipeline_case(a, ts, k):
    cfg = KernelConfig(tilesize=ts, splitk=k)
    m = DenseMatrix.from_array(a)
    pm = pad_to_tiles(m, ts)
    N = pm.rows // ts
    work = pm.copy()
    tau = TauStore(ts, N, m.precision.compute_dtype)
    with ParallelBackend(1) as be:
        band = banddiag(work, tau, N, cfg, be)
        bid = band_to_bidiagonal(band)
        vals = svdvals(m, cfg, be)
    return dict(a=np.asarray(a), ts=np.int64(ts), splitk=np.int64(k), band=np.asfortranarray(work.array),
                tau=np.asfortranarray(tau.values), d=bid.d, e=bid.e, vals=vals)


def main():
    cases = {}
    for dt in (np.float64, np.float32, np.float16):
        for ts, k in ((8, 2), (8, 3), (16, 5), (32, 8), (32, 32), (64, 16)):
            rng = np.random.default_rng(3000 + 17 * ts + k)
            a = rng.standard_normal((ts, ts)).astype(dt)
            mm = DenseMatrix.from_array(a)
            tau = np.zeros(ts, mm.precision.compute_dtype)
            B.geqrt(mm.view(), tau, KernelConfig(tilesize=ts, splitk=k), ParallelBackend(1))
            cases[f"splitk_geqrt_{np.dtype(dt).name}_ts{ts}_k{k}"] = dict(
                a=a, splitk=np.int64(k), out=np.asfortranarray(mm.array), tau=tau)
    for dt, n, ts, k in ((np.float64, 64, 16, 3), (np.float32, 96, 32, 8), (np.float16, 40, 8, 2),
                         (np.float32, 50, 16, 5), (np.float64, 32, 8, 8)):
        rng = np.random.default_rng(4000 + n + ts + k)
        a = rng.standard_normal((n, n)).astype(dt)
        cases[f"splitk_pipe_{np.dtype(dt).name}_n{n}_ts{ts}_k{k}"] = pipeline_case(a, ts, k)
    for name, v in cases.items():
        np.savez_compressed(os.path.join(OUT, name + ".npz"), **v)
    print(f"wrote {len(cases)} split-K fixtures, reference bandsvd {B.__version__}")


if __name__ == "__main__":
    sys.exit(main())
