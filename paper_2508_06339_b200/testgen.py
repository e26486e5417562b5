"""Test-matrix generation for the accuracy and benchmark harness (SURVEY.md
8(f) row 3): the reference's `bandsvd.testgen` interface (testgen.py:27-169)
with a GPU path for the large configurations.

* CPU path -- `SeededRng`, `SpectrumSpec.values`, `random_orthogonal`,
  `make_test_matrix` and `max_relative_error` restate testgen.py:27-98 and
  :160-169 step for step (numpy Philox-4x64 keyed on (seed, stream), QR of a
  Gaussian with the R-diagonal signs absorbed), so a given (seed, stream)
  yields the reference's matrix bit for bit (tests/test_testgen.py checks it
  against tests/golden/testgen_*.npz, produced by the reference itself).
* GPU path (`device=`) -- the same construction on the device: Gaussian
  from a torch Philox generator seeded with (seed, stream), Householder QR
  and the products through torch (cuSOLVER / cuBLAS: this is input
  generation, not the hot path).  Statistically identical to the CPU path,
  not bit-identical (a different Philox stream layout); at n = 16384 it
  takes seconds where host QR takes minutes and 8+ GiB.
* `SpectrumSpec` adds one kind to the reference's three: "graded", the
  cond-1e8 spectrum of configs[2] (sigma_i = 10^(-8 (i-1)/(n-1))).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DegenerateInputError, ShapeError
from .matrix import DenseMatrix
from .precision import FP64, Precision

SPECTRUM_KINDS = ("arithmetic", "logarithmic", "quarter_circle", "graded")


class SeededRng:
    """Counter-based generator (numpy Philox-4x64) keyed on a 64-bit seed and
    a stream tag (testgen.py:27-43): identical keys give bit-identical streams."""

    def __init__(self, seed: int, stream: int = 0):
        self.seed = int(seed)
        self.stream = int(stream)
        key = np.array([self.seed % (1 << 64), self.stream % (1 << 64)], dtype=np.uint64)
        self._gen = np.random.Generator(np.random.Philox(key=key))

    def standard_normal(self, shape):
        return self._gen.standard_normal(shape)

    def uniform(self, size):
        return self._gen.random(size)

    def torch_generator(self, device):
        """A device generator derived from (seed, stream) for the GPU path."""
        import torch
        g = torch.Generator(device=device)
        g.manual_seed((self.seed * 0x9E3779B97F4A7C15 + self.stream) % (1 << 63))
        return g


@dataclass(frozen=True)
class SpectrumSpec:
    """Singular value distribution on [0, 1] (testgen.py:46-74)."""
    kind: str
    n: int

    def __post_init__(self):
        if self.kind not in SPECTRUM_KINDS:
            raise ValueError(f"unknown spectrum kind {self.kind!r}, expected one of {SPECTRUM_KINDS}")
        if self.n < 1:
            raise ShapeError(f"spectrum size must be >= 1, got {self.n}")

    def values(self, rng: SeededRng | None = None) -> np.ndarray:
        """The sigma vector, descending, float64."""
        n = self.n
        if self.kind == "arithmetic":
            return (np.arange(n, 0, -1, dtype=np.float64)) / n
        if self.kind == "logarithmic":
            if n == 1:
                return np.ones(1)
            expo = -6.0 * (n - np.arange(1, n + 1, dtype=np.float64)) / (n - 1)
            return np.sort(10.0 ** expo)[::-1].copy()
        if self.kind == "graded":
            if n == 1:
                return np.ones(1)
            return 10.0 ** (-8.0 * np.arange(n, dtype=np.float64) / (n - 1))
        if rng is None:
            raise ValueError("quarter_circle sampling needs an rng")
        out = np.empty(0)
        while out.size < n:
            cand = rng.uniform(4 * n)
            keep = rng.uniform(4 * n) <= np.sqrt(1.0 - cand * cand)
            out = np.concatenate([out, cand[keep]])
        return np.sort(out[:n])[::-1].copy()


def random_orthogonal(n: int, rng: SeededRng, device=None):
    """Haar-distributed orthogonal matrix (testgen.py:77-87): QR of an iid
    standard-normal matrix with the R diagonal's signs absorbed into Q.
    device=None: numpy on the host (bit-compatible with the reference);
    otherwise a float64 torch tensor built on that device."""
    if n < 1:
        raise ShapeError(f"size must be >= 1, got {n}")
    if device is None:
        g = rng.standard_normal((n, n))
        q, r = np.linalg.qr(g)
        d = np.sign(np.diag(r))
        d[d == 0] = 1.0
        return q * d
    import torch
    g = torch.randn((n, n), generator=rng.torch_generator(device), device=device, dtype=torch.float64)
    q, r = torch.linalg.qr(g)
    d = torch.sign(torch.diagonal(r))
    d[d == 0] = 1.0
    return q * d


def make_test_matrix(spec: SpectrumSpec, rng: SeededRng, precision: Precision = FP64, device=None):
    """(matrix, known values): A = U' diag(sigma) V in the requested precision
    (testgen.py:90-98); the comparison target stays the float64 sigma.
    device=None returns a DenseMatrix (host); otherwise a torch tensor of the
    storage dtype on `device`, ready for svdvals without a host round trip."""
    sigma = spec.values(rng)
    if device is None:
        u = random_orthogonal(spec.n, rng)
        v = random_orthogonal(spec.n, rng)
        a = (u * sigma) @ v
        return DenseMatrix.from_array(a, precision), sigma
    import torch
    u = random_orthogonal(spec.n, rng, device)
    v = random_orthogonal(spec.n, rng, device)
    s = torch.from_numpy(sigma).to(device)
    a = (u * s) @ v
    tdt = {8: torch.float64, 4: torch.float32, 2: torch.float16}[np.dtype(precision.storage_dtype).itemsize]
    return a.to(tdt), sigma


def max_relative_error(computed, reference) -> float:
    """Relative Frobenius-norm error between value vectors (testgen.py:160-169)."""
    c = np.asarray(computed, dtype=np.float64)
    r = np.asarray(reference, dtype=np.float64)
    if c.shape != r.shape:
        raise ShapeError(f"value vectors differ in length: {c.shape} vs {r.shape}")
    denom = float(np.sqrt(np.sum(r * r)))
    if denom == 0.0:
        raise DegenerateInputError("all-zero reference values")
    return float(np.sqrt(np.sum((c - r) ** 2)) / denom)
