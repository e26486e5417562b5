"""TEST INFRASTRUCTURE ONLY -- ctypes front-end of the C restatement of the
reference `bandsvd` path (oracle/bsvd_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module; the product package never does.  Each function mirrors
the reference function it restates (file:line in the C source):

* ``svdvals``      secondstage.py:510-542  (pad -> banddiag -> chase -> bdsqr)
* ``banddiag``     bandreduce.py:91-120
* ``geqrt``        kernels.py:205-230

Precision codes follow the BSVD file format (matrix.py:18):
1 = fp64, 2 = fp32, 3 = fp16-storage (fp32 compute).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

PREC_OF_DTYPE = {np.dtype(np.float64): 1, np.dtype(np.float32): 2, np.dtype(np.float16): 3}
COMPUTE_OF_STORAGE = {np.dtype(np.float64): np.dtype(np.float64),
                      np.dtype(np.float32): np.dtype(np.float32),
                      np.dtype(np.float16): np.dtype(np.float32)}


def build() -> str:
    """Compile liboracle.so in place (needs gcc; the GPU box uses the copy
    built here, which travels with the snapshot)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        vp, i64, i32, dp = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        L.oracle_svdvals.argtypes = [i32, vp, i64, i32, dp, vp, dp, dp]
        L.oracle_svdvals.restype = i32
        L.oracle_banddiag.argtypes = [i32, vp, i32, i32, vp]
        L.oracle_banddiag.restype = None
        L.oracle_geqrt.argtypes = [i32, vp, i32, vp]
        L.oracle_geqrt.restype = None
        L.oracle_geqrt_splitk.argtypes = [i32, vp, i32, vp, i32]
        L.oracle_geqrt_splitk.restype = None
        L.oracle_svdvals_splitk.argtypes = [i32, vp, i64, i32, dp, vp, dp, dp, i32]
        L.oracle_svdvals_splitk.restype = i32
        L.oracle_banddiag_splitk.argtypes = [i32, vp, i32, i32, vp, i32]
        L.oracle_banddiag_splitk.restype = None
        L.oracle_bidiagonal_values.argtypes = [dp, dp, i64]
        L.oracle_bidiagonal_values.restype = i32
        L.oracle_num_threads.restype = i32
        L.oracle_set_num_threads.argtypes = [i32]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def set_num_threads(n: int) -> None:
    lib().oracle_set_num_threads(int(n))


def default_tilesize(n: int) -> int:
    """kernels.py:57-64 `KernelConfig.for_size`."""
    ts = 4
    while ts < 128 and ts * 8 < n:
        ts *= 2
    return ts


def svdvals(a, ts: int | None = None, return_stages: bool = False, splitk: int = 1):
    """All singular values, descending, in the compute dtype (FP16 -> float32).

    ``a`` is a square array whose dtype selects the precision (float64 /
    float32 / float16; anything else is converted to float64 like
    DenseMatrix.from_array, matrix.py:56-67).  With ``return_stages`` also
    returns the padded stage-1 band (column-major storage dtype, as a 2-D
    Fortran view) and the stage-2 bidiagonal (d, e) widened to float64.
    """
    a = np.asarray(a)
    if a.dtype not in PREC_OF_DTYPE:
        a = a.astype(np.float64)
    if a.ndim != 2 or a.shape[0] != a.shape[1] or a.shape[0] < 1:
        raise ValueError(f"expected a non-empty square matrix, got {a.shape}")
    if not np.all(np.isfinite(a.astype(np.float64))):
        raise ValueError("input contains NaN or Inf entries")
    n = a.shape[0]
    ts = ts or default_tilesize(n)
    N = max(1, -(-n // ts))
    npad = N * ts
    src = np.asfortranarray(a)
    vals = np.zeros(n, np.float64)
    band = np.zeros(npad * npad, a.dtype) if return_stages else None
    d = np.zeros(npad, np.float64) if return_stages else None
    e = np.zeros(max(npad - 1, 1), np.float64) if return_stages else None
    rc = lib().oracle_svdvals_splitk(PREC_OF_DTYPE[a.dtype], _ptr(src), n, ts, _ptr(vals),
                                     _ptr(band) if band is not None else None,
                                     _ptr(d) if d is not None else None,
                                     _ptr(e) if e is not None else None, int(splitk))
    if rc != 0:
        raise ArithmeticError("bidiagonal value iteration exceeded its sweep budget")
    out = vals.astype(COMPUTE_OF_STORAGE[a.dtype])
    if return_stages:
        return out, band.reshape((npad, npad), order="F"), d, e[:npad - 1]
    return out


def banddiag(a_padded_colmajor: np.ndarray, ts: int, splitk: int = 1):
    """Stage 1 in place on a padded Fortran-order square; returns the tau store
    (splitk > 1: the split-K panel kernels, kernels.py:233-361)."""
    a = a_padded_colmajor
    assert a.flags.f_contiguous and a.shape[0] == a.shape[1] and a.shape[0] % ts == 0
    N = a.shape[0] // ts
    tau = np.zeros(ts * 2 * N * N, COMPUTE_OF_STORAGE[a.dtype])
    lib().oracle_banddiag_splitk(PREC_OF_DTYPE[a.dtype], _ptr(a), N, ts, _ptr(tau), int(splitk))
    return tau.reshape((ts, 2 * N * N), order="F")


def geqrt(tile: np.ndarray, splitk: int = 1):
    """Tile QR in place (Fortran-order ts x ts); returns tau (compute dtype).
    splitk > 1: geqrt_splitk (kernels.py:459-470)."""
    assert tile.flags.f_contiguous
    ts = tile.shape[0]
    tau = np.zeros(ts, COMPUTE_OF_STORAGE[tile.dtype])
    lib().oracle_geqrt_splitk(PREC_OF_DTYPE[tile.dtype], _ptr(tile), ts, _ptr(tau), int(splitk))
    return tau


def bidiagonal_values(d, e):
    """secondstage.py:473-507 on float64 copies; descending float64."""
    d = np.array(d, np.float64)
    e = np.array(e, np.float64)
    if d.size > 1:
        rc = lib().oracle_bidiagonal_values(_ptr(d), _ptr(e), d.size)
    else:
        d = np.abs(d)
        rc = 0
    if rc != 0:
        raise ArithmeticError("bidiagonal value iteration exceeded its sweep budget")
    return d
