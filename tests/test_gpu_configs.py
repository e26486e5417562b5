"""Parity at the BASELINE.json configs, in the driver-run GPU suite.

Every case checks BOTH metrics of tests/tolerances.py (max |dsigma| / sigma_max
and the reference's normwise max_relative_error, testgen.py:160-169) against
the north star's k*n*eps*||A||_2 bound:

* C1  1024^2 FP32, ts = 32: the pinned C oracle (bit-exact restatement of the
  reference) on the same input;
* C2  8192^2 FP32, default tiles (for_size -> 128): fp64 SVD (cuSOLVER) of the
  same stored input, plus a 2048^2 sample of the same generator against the
  oracle;
* C3  16384^2 FP64, graded spectrum cond 1e8 (sigma_i = 10^(-8 i/(n-1)), Haar
  U, V): the known sigma;
* C4  8192^2 FP16 storage: fp64 SVD of the fp16-rounded input, eps16 bound;
* C5  4096 x 512^2 FP32, ts = 64 (for_size(512)): eight members against the
  oracle, the rest against fp64 cuSOLVER;
* the KernelConfig knobs the fast path accepts (splitk, colperblock < ts), the
  tree stage 1 (BSVD_FLAT=0) and the opt-in tensor-core update (BSVD_TC=1)
  against the oracle;
* run-to-run determinism of the whole pipeline (
  test_acceptance.py:137-181 holds the reference to bitwise reproducibility).
"""
import numpy as np
import pytest

from tolerances import assert_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2508_06339_b200 as P
    return P


@pytest.fixture(scope="module")
def torch():
    import torch
    return torch


def _gauss(torch, n, seed, dtype=None):
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = torch.randn((n, n), generator=g, device="cuda", dtype=torch.float32)
    return a if dtype is None else a.to(dtype)


def _ref_svdvals(torch, a):
    """fp64 cuSOLVER singular values of the stored input."""
    return torch.linalg.svdvals(a.double()).cpu().numpy()


def test_c1_1024_fp32_ts32_vs_oracle(P, oracle):
    a = np.random.default_rng(0xC1).standard_normal((1024, 1024)).astype(np.float32)
    got = P.svdvals(a, P.KernelConfig(tilesize=32))
    assert got.dtype == np.float32 and got.shape == (1024,)
    assert_close(got, oracle.svdvals(a, 32), np.float32, 1024, what="C1 vs oracle")
    want = np.linalg.svd(a.astype(np.float64), compute_uv=False)
    assert_close(got, want, np.float32, 1024, what="C1 vs LAPACK")


def test_c2_8192_fp32_default_tiles(P, torch):
    a = _gauss(torch, 8192, 0xC2)
    got = P.svdvals(a)                         # cfg=None -> for_size(8192) -> ts 128
    assert got.is_cuda and got.dtype == torch.float32
    assert bool(torch.all(got[:-1] >= got[1:]))
    assert_close(got.double().cpu().numpy(), _ref_svdvals(torch, a), np.float32, 8192, what="C2")


def test_c2_sample_2048_vs_oracle(P, torch, oracle):
    a = _gauss(torch, 2048, 0xC2)
    got = P.svdvals(a).cpu().numpy()
    # a row-major device tensor is read as A^T: the oracle gets the same matrix
    assert_close(got, oracle.svdvals(a.cpu().numpy().T.copy(), 128), np.float32, 2048,
                 what="C2 2048 sample vs oracle")


def _graded(torch, n, cond, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    sig = torch.logspace(0, -np.log10(cond), n, dtype=torch.float64, device="cuda")
    u, _ = torch.linalg.qr(torch.randn(n, n, generator=g, dtype=torch.float64, device="cuda"))
    v, _ = torch.linalg.qr(torch.randn(n, n, generator=g, dtype=torch.float64, device="cuda"))
    a = (u * sig) @ v.T
    del u, v
    return a, sig.cpu().numpy()


def test_c3_16384_fp64_graded_known_sigma(P, torch):
    a, sig = _graded(torch, 16384, 1e8, 3)
    got = P.svdvals(a)
    assert got.dtype == torch.float64
    assert_close(got.cpu().numpy(), sig, np.float64, 16384, what="C3 vs known sigma")
    del a
    torch.cuda.empty_cache()


def test_c4_8192_fp16_storage(P, torch):
    a = _gauss(torch, 8192, 0xC4, torch.float16)
    got = P.svdvals(a)
    assert got.dtype == torch.float32           # FP16 computes (and returns) in fp32
    assert_close(got.double().cpu().numpy(), _ref_svdvals(torch, a), np.float16, 8192, what="C4")


def test_c5_batch_4096x512_ts64(P, torch, oracle):
    B, n = 4096, 512
    g = torch.Generator(device="cuda").manual_seed(0xC5)
    x = torch.randn((B, n, n), generator=g, device="cuda")
    got = P.svdvals_batched(x)                  # cfg=None -> for_size(512) -> ts 64
    assert got.shape == (B, n)
    idx = [0, 1, 2, 511, 2048, 3000, 4094, 4095]
    for i in idx:   # the batch reads each row-major member as its transpose
        want = oracle.svdvals(x[i].cpu().numpy().T.copy(), 64)
        assert_close(got[i].cpu().numpy(), want, np.float32, n, what=f"C5 member {i} vs oracle")
    sample = list(range(0, B, 257))
    ref = torch.linalg.svdvals(x[sample].double()).cpu().numpy()
    for j, i in enumerate(sample):
        assert_close(got[i].double().cpu().numpy(), ref[j], np.float32, n, what=f"C5 member {i}")


@pytest.mark.parametrize("splitk,cpb", [(2, None), (8, None), (1, 32), (4, 16)])
def test_fast_path_config_knobs(P, oracle, splitk, cpb):
    """splitk / colperblock are validated like the reference (kernels.py:42-55)
    and leave the fast path's values within the bound."""
    n, ts = 768, 64
    a = np.random.default_rng(splitk * 100 + (cpb or 0)).standard_normal((n, n)).astype(np.float32)
    cfg = P.KernelConfig(tilesize=ts, splitk=splitk, colperblock=cpb or ts)
    assert_close(P.svdvals(a, cfg), oracle.svdvals(a, ts), np.float32, n, what=f"splitk={splitk} cpb={cpb}")


@pytest.mark.parametrize("dtype", [np.float32, np.float16])
@pytest.mark.parametrize("n,ts", [(1024, 128), (640, 64), (1100, 128)])
def test_tree_stage1_vs_oracle(P, oracle, monkeypatch, dtype, n, ts):
    """The tree stage 1 (two-tile leaves + TT nodes) that FP32/FP16 ran before
    the flat cluster panel became the default for ts in {64, 128}."""
    monkeypatch.setenv("BSVD_FLAT", "0")
    a = np.random.default_rng(n + ts).standard_normal((n, n)).astype(dtype)
    assert_close(P.svdvals(a, P.KernelConfig(tilesize=ts)), oracle.svdvals(a, ts), dtype, n,
                 what=f"tree n={n} ts={ts}")


@pytest.mark.parametrize("n", [512, 1024])
def test_tc_update_path_vs_oracle(P, oracle, monkeypatch, n):
    """The opt-in tcgen05 3xTF32 trailing update of the tree stage 1."""
    monkeypatch.setenv("BSVD_FLAT", "0")
    monkeypatch.setenv("BSVD_TC", "1")
    a = np.random.default_rng(n).standard_normal((n, n)).astype(np.float32)
    assert_close(P.svdvals(a, P.KernelConfig(tilesize=128)), oracle.svdvals(a, 128), np.float32, n,
                 what=f"tc n={n}")


@pytest.mark.parametrize("n,ts,dtype", [(2048, 128, "float32"), (1024, 32, "float32"),
                                        (512, 64, "float16"), (768, 128, "float64")])
def test_run_to_run_deterministic(P, torch, n, ts, dtype):
    """Fixed reduction orders everywhere (no float atomics): two runs of the
    same input give the same bits."""
    a = _gauss(torch, n, 99, getattr(torch, dtype))
    cfg = P.KernelConfig(tilesize=ts)
    first = P.svdvals(a, cfg).cpu().numpy()
    for _ in range(2):
        again = P.svdvals(a, cfg).cpu().numpy()
        assert np.array_equal(first.view(np.uint8), again.view(np.uint8))
    b = torch.stack([a, a.flip(0)])
    bat = P.svdvals_batched(b, cfg).cpu().numpy()
    assert np.array_equal(bat, P.svdvals_batched(b, cfg).cpu().numpy())


@pytest.mark.parametrize("dtype", [np.float32, np.float16])
@pytest.mark.parametrize("case", ["zero", "identity", "rank1", "tiny", "huge", "graded"])
def test_tensor_core_path_edge_inputs(P, oracle, dtype, case):
    """ts = 128 FP32 / FP16 storage runs the tcgen05 update path: degenerate
    and badly scaled inputs (exact zeros, identity, rank one, 1e-30 / 1e30
    scaling within the storage range, a graded spectrum) give the oracle's
    values within the bound."""
    n = 384
    rng = np.random.default_rng(hash(case) % 1000)
    if case == "zero":
        a = np.zeros((n, n))
    elif case == "identity":
        a = np.eye(n)
    elif case == "rank1":
        a = np.outer(rng.standard_normal(n), rng.standard_normal(n))
    elif case == "tiny":
        a = rng.standard_normal((n, n)) * (1e-30 if dtype == np.float32 else 1e-3)
    elif case == "huge":
        a = rng.standard_normal((n, n)) * (1e30 if dtype == np.float32 else 1e3)
    else:
        u, _ = np.linalg.qr(rng.standard_normal((n, n)))
        v, _ = np.linalg.qr(rng.standard_normal((n, n)))
        a = (u * np.logspace(0, -6, n)) @ v.T
    a = a.astype(dtype)
    got = P.svdvals(a, P.KernelConfig(tilesize=128))
    if case == "zero":
        assert not np.any(got)
        return
    if case == "identity":
        assert np.array_equal(got, np.ones(n, np.float32))
        return
    want = np.linalg.svd(a.astype(np.float64), compute_uv=False)
    assert_close(got, want, dtype, n, what=f"{case} {np.dtype(dtype).name}")


@pytest.mark.parametrize("dtype", [np.float32, np.float16])
def test_tensor_core_path_batched(P, oracle, dtype):
    """Batches on the ts = 128 tensor-core path (blockIdx.z = member, one TMA
    map with a batch dimension), ragged n (zero padding to 128)."""
    rng = np.random.default_rng(8)
    a = rng.standard_normal((3, 300, 300)).astype(dtype)
    got = P.svdvals_batched(a, P.KernelConfig(tilesize=128))
    for i in range(3):
        assert_close(got[i], oracle.svdvals(a[i].T.copy(), 128), dtype, 300, what=f"member {i}")


@pytest.mark.parametrize("n,ts,dtype", [(1024, 128, "float32"), (1000, 64, "float32"),
                                        (777, 32, "float16"), (2048, 128, "float32")])
def test_chase_edge_mailbox_bitwise(P, torch, monkeypatch, n, ts, dtype):
    """The fp32 cluster chase hands the edges to the next sweep through the tagged
    mailbox; the edge-flag protocol (BSVD_CHASE_MBOX=0) moves the same values, so
    both give the same bits."""
    a = _gauss(torch, n, 7 + n, getattr(torch, dtype))
    cfg = P.KernelConfig(tilesize=ts)
    got = P.svdvals(a, cfg).cpu().numpy()
    monkeypatch.setenv("BSVD_CHASE_MBOX", "0")
    ref = P.svdvals(a, cfg).cpu().numpy()
    assert np.array_equal(got, ref), f"mailbox vs flags differ: n={n} ts={ts} {dtype}"


@pytest.mark.parametrize("n,ts", [(640, 32), (900, 64)])
def test_chase_wide_tile_on_narrow_band_vs_oracle(P, oracle, monkeypatch, n, ts):
    """Narrow bands run 32 / 64-wide chase tiles; the 128-wide tile
    (BSVD_CHASE_BK=128) on the same band stays within tolerance of the oracle."""
    a = np.random.default_rng(n).standard_normal((n, n)).astype(np.float32)
    want = oracle.svdvals(a, ts)
    assert_close(P.svdvals(a, P.KernelConfig(tilesize=ts)), want, np.float32, n, what=f"tile n={n} ts={ts}")
    monkeypatch.setenv("BSVD_CHASE_BK", "128")
    assert_close(P.svdvals(a, P.KernelConfig(tilesize=ts)), want, np.float32, n, what=f"tile128 n={n} ts={ts}")
