"""The C oracle (oracle/bsvd_oracle.c) reproduces the REFERENCE bit-for-bit
on the golden vectors generated from the reference itself
(scripts/make_golden.py).  CPU only."""
import numpy as np
import pytest

from conftest import golden_names, load_golden, same_bits


@pytest.mark.parametrize("name", golden_names("pipe_"))
def test_pipeline_bitwise(oracle, name):
    g = load_golden(name)
    vals, band, d, e = oracle.svdvals(g["a"], int(g["ts"]), return_stages=True)
    assert same_bits(band, g["band"]), "stage-1 band differs"
    assert np.array_equal(d, g["d"].astype(np.float64)), "stage-2 d differs"
    assert np.array_equal(e, g["e"].astype(np.float64)), "stage-2 e differs"
    assert vals.dtype == g["vals"].dtype
    assert np.array_equal(vals, g["vals"]), "values differ"


@pytest.mark.parametrize("name", golden_names("geqrt_"))
def test_geqrt_bitwise(oracle, name):
    g = load_golden(name)
    tile = np.asfortranarray(g["a"].copy())
    tau = oracle.geqrt(tile)
    assert same_bits(tile, g["out"])
    assert np.array_equal(tau.astype(g["tau"].dtype), g["tau"])


@pytest.mark.parametrize("name", golden_names("bidiag_"))
def test_bidiagonal_values_bitwise(oracle, name):
    g = load_golden(name)
    got = oracle.bidiagonal_values(g["d"], g["e"])
    assert np.array_equal(got, g["vals"])


def test_known_answers(oracle):
    assert np.array_equal(oracle.svdvals(np.diag([3.0, 2.0, 1.0])), [3.0, 2.0, 1.0])
    gold = oracle.bidiagonal_values([1.0, 1.0], [1.0])
    assert np.allclose(gold, [(1 + 5 ** 0.5) / 2, (5 ** 0.5 - 1) / 2], rtol=1e-14)


def test_scaling_equivariance(oracle):
    a = np.random.default_rng(10).standard_normal((24, 24))
    assert np.array_equal(oracle.svdvals(4.0 * a), 4.0 * oracle.svdvals(a))


def test_threads_do_not_change_bits(oracle):
    a = np.random.default_rng(3).standard_normal((96, 96)).astype(np.float32)
    n0 = oracle.num_threads()
    oracle.set_num_threads(1)
    v1 = oracle.svdvals(a, 16)
    oracle.set_num_threads(max(n0, 2))
    v2 = oracle.svdvals(a, 16)
    oracle.set_num_threads(n0)
    assert np.array_equal(v1, v2)


# ---- split-K panels (kernels.py:233-361; scripts/make_golden_splitk.py) ----

@pytest.mark.parametrize("name", golden_names("splitk_geqrt_"))
def test_geqrt_splitk_bitwise(oracle, name):
    g = load_golden(name)
    tile = np.asfortranarray(g["a"].copy())
    tau = oracle.geqrt(tile, splitk=int(g["splitk"]))
    assert same_bits(tile, g["out"])
    assert np.array_equal(tau.astype(g["tau"].dtype), g["tau"])


@pytest.mark.parametrize("name", golden_names("splitk_pipe_"))
def test_pipeline_splitk_bitwise(oracle, name):
    g = load_golden(name)
    vals, band, d, e = oracle.svdvals(g["a"], int(g["ts"]), return_stages=True, splitk=int(g["splitk"]))
    assert same_bits(band, g["band"]), "stage-1 band differs"
    assert np.array_equal(d, g["d"].astype(np.float64)), "stage-2 d differs"
    assert np.array_equal(vals, g["vals"]), "values differ"


def test_splitk_changes_the_arithmetic(oracle):
    """The split-K order is a different rounding sequence: the fixtures are
    not the splitk = 1 bytes (so the tests above pin real behaviour)."""
    differs = 0
    for name in golden_names("splitk_geqrt_"):
        g = load_golden(name)
        tile = np.asfortranarray(g["a"].copy())
        oracle.geqrt(tile)
        differs += not same_bits(tile, g["out"])
    assert differs >= len(golden_names("splitk_geqrt_")) // 2
