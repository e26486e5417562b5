"""Generate tests/golden/*.npz from the REFERENCE implementation itself.

Run in the build container, where the read-only reference is importable:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python scripts/make_golden.py

The fixtures pin both the C oracle (tests/test_oracle_pinning.py, bit-exact)
and the B200 engine (tests/test_gpu_parity.py, bit-exact for the faithful
stage-1 kernels, tolerance-based for the full pipeline).  Nothing at test
time reads /root/reference; only these committed arrays travel.

Cases mirror the reference's own tests: bitwise GEQRT transcription
(test_kernels.py:69-76), identity/zero tiles (:58-67), [I; I] stack
(:133-141), fused-chain driver (test_bandreduce.py), stage-2/3 known answers
(test_secondstage.py:29-153), scaling equivariance (:170-180), padding
(:189-195) and the FP16-storage pipeline (:210-216).
"""
from __future__ import annotations

import os
import sys

import numpy as np

import bandsvd as B
from bandsvd import (BidiagonalMatrix, DenseMatrix, KernelConfig, ParallelBackend,
                     ReferenceBackend, SeededRng, SpectrumSpec, TauStore,
                     band_to_bidiagonal, banddiag, bidiagonal_values,
                     make_test_matrix, svdvals)
from bandsvd.matrix import pad_to_tiles

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "tests", "golden")


def pipeline_case(a, ts):
    """Reference stage outputs for one input (storage dtype preserved)."""
    m = DenseMatrix.from_array(a)
    pm = pad_to_tiles(m, ts)
    N = pm.rows // ts
    work = pm.copy()
    tau = TauStore(ts, N, m.precision.compute_dtype)
    with ParallelBackend(1) as be:
        band = banddiag(work, tau, N, KernelConfig(tilesize=ts), be)
        bid = band_to_bidiagonal(band)
        vals = svdvals(m, KernelConfig(tilesize=ts), be)
    return dict(a=np.asarray(a), ts=np.int64(ts), band=np.asfortranarray(work.array),
                tau=np.asfortranarray(tau.values), d=bid.d, e=bid.e, vals=vals)


def main():
    os.makedirs(OUT, exist_ok=True)
    cases = {}
    # --- end-to-end pipeline cases, three precisions ---------------------
    for dt in (np.float64, np.float32, np.float16):
        for n, ts in ((8, 4), (13, 4), (32, 8), (64, 16), (96, 32)):
            rng = np.random.default_rng(1000 + 7 * n + ts)
            a = rng.standard_normal((n, n)).astype(dt)
            cases[f"pipe_{np.dtype(dt).name}_n{n}_ts{ts}"] = pipeline_case(a, ts)
    # Gaussian from the reference's own bench generator (bench.py:48-50)
    g = SeededRng(0, stream=0xBE7C).standard_normal((128, 128))
    cases["pipe_bench_gauss_float32_n128_ts32"] = pipeline_case(g.astype(np.float32), 32)
    # known-spectrum matrices (testgen.py:77-98)
    m, sigma = make_test_matrix(SpectrumSpec("logarithmic", 64), SeededRng(7))
    c = pipeline_case(m.array.copy(), 16)
    c["sigma"] = sigma
    cases["pipe_logspec_float64_n64_ts16"] = c
    m, sigma = make_test_matrix(SpectrumSpec("arithmetic", 128), SeededRng(123))
    c = pipeline_case(m.array.copy(), 32)
    c["sigma"] = sigma
    cases["pipe_arith_float64_n128_ts32"] = c
    # A1 landmine: absolute 10*eps reflector guard on tiny-scaled input
    a = np.random.default_rng(5).standard_normal((64, 64))
    cases["pipe_scaled1e-6_float32_n64_ts16"] = pipeline_case((a * 1e-6).astype(np.float32), 16)
    # degenerate inputs (test_acceptance.py:187-201)
    cases["pipe_zero_float64_n16_ts4"] = pipeline_case(np.zeros((16, 16)), 4)
    cases["pipe_identity_float64_n16_ts4"] = pipeline_case(np.eye(16), 4)
    u = np.random.default_rng(9).standard_normal(24)
    v = np.random.default_rng(10).standard_normal(24)
    cases["pipe_rank1_float64_n24_ts8"] = pipeline_case(np.outer(u, v), 8)
    cases["pipe_diag321_float64_n3_ts4"] = pipeline_case(np.diag([3.0, 2.0, 1.0]), 4)
    cases["pipe_perm_float64_n2_ts4"] = pipeline_case(np.array([[0.0, 1.0], [1.0, 0.0]]), 4)

    # --- kernel-level: GEQRT tiles (kernels.py:205-230) -------------------
    for dt in (np.float64, np.float32, np.float16):
        for ts in (4, 8, 16, 32, 64, 128):
            rng = np.random.default_rng(2000 + ts)
            a = rng.standard_normal((ts, ts)).astype(dt)
            mm = DenseMatrix.from_array(a)
            tau = np.zeros(ts, mm.precision.compute_dtype)
            B.geqrt(mm.view(), tau, KernelConfig(tilesize=ts), ParallelBackend(1))
            cases[f"geqrt_{np.dtype(dt).name}_ts{ts}"] = dict(a=a, out=np.asfortranarray(mm.array), tau=tau)
    for name, a in (("identity", np.eye(4)), ("zero", np.zeros((6, 6)))):
        mm = DenseMatrix.from_array(a)
        tau = np.zeros(a.shape[0])
        B.geqrt(mm.view(), tau, KernelConfig(tilesize=a.shape[0]), ReferenceBackend())
        cases[f"geqrt_{name}"] = dict(a=a, out=np.asfortranarray(mm.array), tau=tau)
    # TSQRT [I; I] -> -sqrt(2) I (test_kernels.py:133-141)
    rm, bm = DenseMatrix.from_array(np.eye(4)), DenseMatrix.from_array(np.eye(4))
    tau = np.zeros(4)
    B.tsqrt(rm.view(), bm.view(), tau, KernelConfig(tilesize=4), ReferenceBackend())
    cases["tsqrt_identity_stack"] = dict(r=np.asfortranarray(rm.array), b=np.asfortranarray(bm.array), tau=tau)

    # --- stage 3 known answers (test_secondstage.py:104-153) -------------
    bid_cases = {
        "golden": (np.array([1.0, 1.0]), np.array([1.0])),
        "zero_diag": (np.array([1.0, 0.0]), np.array([0.0])),
        "zero_diag_coupled": (np.array([0.0, 1.0, 2.0]), np.array([1.0, 1.0])),
        "diag321": (np.array([3.0, 2.0, 1.0]), np.zeros(2)),
    }
    rng = np.random.default_rng(6)
    for n in (2, 7, 33, 200):
        bid_cases[f"random{n}"] = (rng.standard_normal(n), rng.standard_normal(n - 1))
    for k, (d, e) in bid_cases.items():
        vals = bidiagonal_values(BidiagonalMatrix(d.copy(), e.copy()))
        cases[f"bidiag_{k}"] = dict(d=d, e=e, vals=vals)

    for k, v in cases.items():
        np.savez_compressed(os.path.join(OUT, k + ".npz"), **v)
    total = sum(os.path.getsize(os.path.join(OUT, f)) for f in os.listdir(OUT))
    print(f"wrote {len(cases)} fixtures, {total / 1024:.0f} KiB, reference bandsvd {B.__version__}")


if __name__ == "__main__":
    sys.exit(main())
