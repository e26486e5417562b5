"""The C-ABI library loads and exports every symbol include/bsvd.h declares;
host-only entry points (no CUDA calls) behave like the reference.  CPU only."""
import ctypes
import os
import re

import pytest

from conftest import ROOT


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "bsvd.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(bsvd_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_2508_06339_b200 import _lib
    L = _lib.load()
    syms = _header_symbols()
    assert len(syms) >= 16
    for s in syms:
        assert hasattr(L, s), f"missing export {s}"
    assert set(syms) == set(_lib.EXPORTS)


def test_validate_config_matches_reference_rules():
    from paper_2508_06339_b200 import _lib
    L = _lib.load()
    ok = lambda ts, cpb, k: L.bsvd_validate_config(ctypes.byref(_lib.BsvdConfig(ts, cpb, k, 1)))
    assert ok(32, 32, 1) == 0
    assert ok(2, 0, 1) == _lib.BSVD_E_CONFIG
    assert ok(256, 0, 1) == _lib.BSVD_E_CONFIG
    assert ok(32, 7, 1) == _lib.BSVD_E_CONFIG
    assert ok(32, 64, 1) == _lib.BSVD_E_CONFIG
    assert ok(64, 0, 64) == _lib.BSVD_E_CONFIG
    assert ok(64, 0, 16) == 0
    assert ok(32, 0, 33) == _lib.BSVD_E_CONFIG
    assert b"tilesize" in (ok(2, 0, 1) and L.bsvd_last_error())


def test_default_tilesize_is_for_size():
    from paper_2508_06339_b200 import KernelConfig, _lib
    L = _lib.load()
    for n in (1, 5, 8, 63, 200, 512, 1024, 4096, 16384):
        assert L.bsvd_default_tilesize(n) == KernelConfig.for_size(n).tilesize


def test_workspace_bytes_monotone():
    from paper_2508_06339_b200 import _lib
    L = _lib.load()
    cfg = _lib.BsvdConfig(128, 0, 1, 1)
    a = L.bsvd_workspace_bytes(2, 1024, 1, ctypes.byref(cfg))
    b = L.bsvd_workspace_bytes(2, 2048, 1, ctypes.byref(cfg))
    c = L.bsvd_workspace_bytes(2, 2048, 4, ctypes.byref(cfg))
    assert 0 < a < b < c
    assert L.bsvd_workspace_bytes(9, 1024, 1, ctypes.byref(cfg)) == 0


def test_kernelconfig_python_mirror():
    from paper_2508_06339_b200 import ConfigError, KernelConfig
    with pytest.raises(ConfigError):
        KernelConfig(tilesize=2)
    with pytest.raises(ConfigError):
        KernelConfig(tilesize=32, colperblock=7)
    with pytest.raises(ConfigError):
        KernelConfig(tilesize=64, splitk=64)
    assert KernelConfig(tilesize=32).colperblock == 32
    assert KernelConfig.for_size(8).tilesize == 4
    assert KernelConfig.for_size(1024).tilesize == 128


def test_product_fails_loudly_without_gpu():
    import torch
    from paper_2508_06339_b200 import DeviceError, svdvals
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(DeviceError):
        svdvals([[1.0, 0.0], [0.0, 1.0]])


def test_product_never_imports_oracle():
    import subprocess
    import sys
    code = ("import sys; import paper_2508_06339_b200 as P; "
            "assert not any(m == 'oracle' or m.startswith('oracle.') for m in sys.modules), sys.modules.keys()")
    subprocess.run([sys.executable, "-c", code], check=True, cwd=ROOT)
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_2508_06339_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", src).replace("oracles", ""), f
