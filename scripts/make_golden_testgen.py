"""Golden vectors for paper_2508_06339_b200.testgen's CPU path, produced by the
REFERENCE's own testgen (testgen.py:27-169).  Run in the build container:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python scripts/make_golden_testgen.py
"""
import os

import numpy as np

from bandsvd import FP32, SeededRng, SpectrumSpec, make_test_matrix
from bandsvd.testgen import max_relative_error, random_orthogonal

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                   "testgen_ref.npz")


def main():
    g = SeededRng(5, stream=3)
    out = {"normal": g.standard_normal((4, 6)), "uniform": g.uniform(10)}
    for kind in ("arithmetic", "logarithmic", "quarter_circle"):
        out[f"spec_{kind}"] = SpectrumSpec(kind, 16).values(SeededRng(2, stream=9))
    out["orth"] = random_orthogonal(12, SeededRng(4, stream=1))
    m, sigma = make_test_matrix(SpectrumSpec("quarter_circle", 20), SeededRng(11, stream=2), FP32)
    out["tm_a"] = m.array.copy()
    out["tm_sigma"] = sigma
    out["mre"] = np.float64(max_relative_error(np.arange(1.0, 6.0), np.arange(1.0, 6.0) + 1e-3))
    np.savez(OUT, **out)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
