"""Parity tolerances.

The north star's bound is k * n * eps * ||A||_2, checked BOTH as the max
absolute error scaled by sigma_max (= ||A||_2) and as the reference's own
normwise metric max_relative_error (testgen.py:160-169).  eps is the compute
unit roundoff (2^-52 / 2^-23); k = 1 (the reference itself sits at k ~ 0.03
for FP32 and ~0.4 for FP64 at n = 1024).  FP16 storage uses the storage eps
2^-10 without the n factor (k * n * eps16 >= 1 is vacuous for n >= 1024;
SURVEY.md 7.4-H7), k = 1.  A floor of 16 eps covers tiny n."""
import numpy as np

EPS = {"float64": 2.0 ** -52, "float32": 2.0 ** -23, "float16": 2.0 ** -10}


def bound(storage_dtype, n, k=1.0):
    name = np.dtype(storage_dtype).name
    if name == "float16":
        return k * EPS[name]
    return k * max(n, 16) * EPS[name]


def errors(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    smax = float(np.max(np.abs(want))) if want.size else 0.0
    if smax == 0.0:
        return float(np.max(np.abs(got))) if got.size else 0.0, 0.0
    abs_rel = float(np.max(np.abs(got - want))) / smax
    normwise = float(np.linalg.norm(got - want) / np.linalg.norm(want))
    return abs_rel, normwise


def assert_close(got, want, storage_dtype, n, k=1.0, what=""):
    tol = bound(storage_dtype, n, k)
    a, nw = errors(got, want)
    assert a <= tol and nw <= tol, f"{what}: max-abs/sigma_max {a:.3e}, normwise {nw:.3e} > tol {tol:.3e}"
    return a, nw
