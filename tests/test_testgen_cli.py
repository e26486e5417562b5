"""Test-matrix generation and the CLI.

CPU: the testgen CPU path reproduces the reference's generators bit for bit
(tests/golden/testgen_ref.npz, made by scripts/make_golden_testgen.py from
the reference itself); CLI parsing, value formatting and the BSVD round trip.
GPU: device-generated known-spectrum matrices through svdvals; the CLI's
svdvals / accuracy / bench commands end to end."""
import io
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import load_golden
from tolerances import assert_close

import paper_2508_06339_b200 as P
from paper_2508_06339_b200 import cli, testgen as T

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_testgen_bitwise_vs_reference():
    g = load_golden("testgen_ref")
    r = T.SeededRng(5, stream=3)
    assert np.array_equal(r.standard_normal((4, 6)), g["normal"])
    assert np.array_equal(r.uniform(10), g["uniform"])
    for kind in ("arithmetic", "logarithmic", "quarter_circle"):
        assert np.array_equal(T.SpectrumSpec(kind, 16).values(T.SeededRng(2, stream=9)), g[f"spec_{kind}"])
    assert np.array_equal(T.random_orthogonal(12, T.SeededRng(4, stream=1)), g["orth"])
    m, sigma = T.make_test_matrix(T.SpectrumSpec("quarter_circle", 20), T.SeededRng(11, stream=2), P.FP32)
    assert np.array_equal(m.array, g["tm_a"]) and np.array_equal(sigma, g["tm_sigma"])
    assert T.max_relative_error(np.arange(1.0, 6.0), np.arange(1.0, 6.0) + 1e-3) == float(g["mre"])


def test_testgen_graded_and_errors():
    s = T.SpectrumSpec("graded", 5).values()
    assert s[0] == 1.0 and abs(s[-1] - 1e-8) < 1e-22 and np.all(np.diff(s) < 0)
    with pytest.raises(ValueError):
        T.SpectrumSpec("bogus", 4)
    with pytest.raises(P.ShapeError):
        T.SpectrumSpec("arithmetic", 0)
    with pytest.raises(P.DegenerateInputError):
        T.max_relative_error(np.zeros(3), np.zeros(3))


def test_cli_formatting_and_parsing():
    assert cli.format_value(np.float32(1.0) / np.float32(3.0)) == "0.333333343"
    assert cli.format_value(np.float64(1.0) / 3.0) == "0.33333333333333331"
    assert cli.parse_int_list("64, 256,") == [64, 256]
    args = cli.build_parser().parse_args(["bench", "--sizes", "1024", "--tilesize", "32"])
    assert cli.config_for(args, 1024).tilesize == 32
    args = cli.build_parser().parse_args(["bench", "--sizes", "8192"])
    assert cli.config_for(args, 8192).tilesize == 128


def test_cli_bad_input_exit_code(tmp_path):
    bad = tmp_path / "bad.bsvd"
    bad.write_bytes(b"NOPE")
    assert cli.main(["svdvals", str(bad)]) == 2


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["arithmetic", "logarithmic", "quarter_circle", "graded"])
def test_device_testgen_through_svdvals(kind):
    import torch
    be = P.B200Backend()
    for prec, dtype in ((P.FP64, np.float64), (P.FP32, np.float32)):
        a, sigma = T.make_test_matrix(T.SpectrumSpec(kind, 256), T.SeededRng(3, stream=1), prec, device=be.device)
        assert a.is_cuda and a.shape == (256, 256)
        got = P.svdvals(a, backend=be).double().cpu().numpy()
        assert_close(got, sigma, dtype, 256, what=f"{kind} {np.dtype(dtype).name}")


@pytest.mark.gpu
def test_cli_end_to_end(tmp_path):
    a = np.random.default_rng(2).standard_normal((40, 40)).astype(np.float32)
    path = tmp_path / "m.bsvd"
    P.write_matrix(P.DenseMatrix.from_array(a), path)
    out = tmp_path / "vals.csv"
    assert cli.main(["svdvals", str(path), "--output", str(out)]) == 0
    vals = np.array([float(x) for x in out.read_text().split()])
    want = np.linalg.svd(a.astype(np.float64), compute_uv=False)
    assert_close(vals, want, np.float32, 40)
    acc = tmp_path / "acc.csv"
    assert cli.main(["accuracy", "--sizes", "64", "--precisions", "fp64,fp32", "--per-distribution", "1",
                     "--output", str(acc)]) == 0
    lines = acc.read_text().split()
    assert lines[0] == "size,fp64,fp32"
    e64, e32 = (float(x) for x in lines[1].split(",")[1:])
    assert e64 < 1e-12 and e32 < 1e-5
    bench = tmp_path / "bench.csv"
    assert cli.main(["bench", "--sizes", "256", "--precision", "fp32", "--batch", "2", "--min-total", "0",
                     "--breakdown", "--output", str(bench)]) == 0
    rows = bench.read_text().split()
    assert rows[0].startswith("size,precision,tilesize") and rows[1].startswith("256,fp32,32")
