"""ctypes binding of libbsvd.so (include/bsvd.h).

The shared library is built in-tree (``paper_2508_06339_b200/lib``) by
``__graft_entry__.build()`` / ``make -C paper_2508_06339_b200/csrc``.  There is
no CPU fallback: if the library is missing or no CUDA device is present,
``lib()`` raises ``DeviceError``.
"""
from __future__ import annotations

import ctypes
import os

from .errors import (ConfigError, ConvergenceError, DeviceError, ShapeError,
                     ValidationError)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libbsvd.so")

BSVD_OK, BSVD_E_SHAPE, BSVD_E_CONFIG, BSVD_E_VALIDATION = 0, 2, 3, 4
BSVD_E_CONVERGENCE, BSVD_E_CUDA, BSVD_E_OOM, BSVD_E_NOTIMPL = 5, 6, 7, 8
STAGE1_TREE, STAGE1_FAITHFUL = 0, 1

# every symbol include/bsvd.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "bsvd_validate_config", "bsvd_default_tilesize", "bsvd_default_options",
    "bsvd_last_error", "bsvd_version", "bsvd_workspace_bytes", "bsvd_svdvals",
    "bsvd_svdvals_ex", "bsvd_svdvals_batched", "bsvd_banddiag",
    "bsvd_band_workspace_bytes", "bsvd_band_to_bidiagonal", "bsvd_bidiagonal_values", "bsvd_geqrt",
    "bsvd_tsqrt_chain", "bsvd_geqrt_splitk", "bsvd_tsqrt_chain_splitk", "bsvd_unmqr", "bsvd_tsmqr_fused", "bsvd_launch_counter",
)


class BsvdConfig(ctypes.Structure):
    _fields_ = [("tilesize", ctypes.c_int32), ("colperblock", ctypes.c_int32),
                ("splitk", ctypes.c_int32), ("fused", ctypes.c_int32)]


class BsvdOptions(ctypes.Structure):
    _fields_ = [("stage1_algo", ctypes.c_int32), ("check_finite", ctypes.c_int32),
                ("reserved", ctypes.c_int32 * 6)]


class BsvdTimers(ctypes.Structure):
    _fields_ = [("panel_s", ctypes.c_double), ("trailing_s", ctypes.c_double),
                ("bidiagonal_s", ctypes.c_double), ("diagonal_s", ctypes.c_double)]


_lib = None


def load(path: str = LIB_PATH):
    """Load the library and declare prototypes (no CUDA calls are made)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise DeviceError(f"libbsvd.so not built at {path}; run __graft_entry__.build()")
    L = ctypes.CDLL(path)
    vp, i64, i32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_size_t
    cfgp, optp, timp = ctypes.POINTER(BsvdConfig), ctypes.POINTER(BsvdOptions), ctypes.POINTER(BsvdTimers)
    dp = ctypes.c_void_p
    proto = {
        "bsvd_validate_config": (i32, [cfgp]),
        "bsvd_default_tilesize": (i32, [i64]),
        "bsvd_default_options": (None, [optp]),
        "bsvd_last_error": (ctypes.c_char_p, []),
        "bsvd_version": (ctypes.c_char_p, []),
        "bsvd_launch_counter": (ctypes.c_uint64, []),
        "bsvd_workspace_bytes": (sz, [i32, i64, i64, cfgp]),
        "bsvd_svdvals": (i32, [vp, i32, i64, i64, cfgp, vp, vp, sz, vp, timp]),
        "bsvd_svdvals_ex": (i32, [vp, i32, i64, i64, cfgp, optp, vp, vp, sz, vp, timp]),
        "bsvd_svdvals_batched": (i32, [vp, i32, i64, i64, i64, i64, cfgp, vp, vp, sz, vp, timp]),
        "bsvd_banddiag": (i32, [vp, i32, i64, cfgp, optp, vp, sz, vp]),
        "bsvd_band_workspace_bytes": (sz, [i64, i32]),
        "bsvd_band_to_bidiagonal": (i32, [vp, i32, i64, i32, dp, dp, vp, sz, vp]),
        "bsvd_bidiagonal_values": (i32, [dp, dp, i64, dp, vp]),
        "bsvd_geqrt": (i32, [vp, i64, i64, i32, i32, vp, vp]),
        "bsvd_tsqrt_chain": (i32, [vp, i64, i64, vp, vp, i32, i32, i32, vp]),
        "bsvd_geqrt_splitk": (i32, [vp, i64, i64, i32, i32, i32, vp, vp]),
        "bsvd_tsqrt_chain_splitk": (i32, [vp, i64, i64, vp, vp, i32, i32, i32, i32, vp]),
        "bsvd_unmqr": (i32, [vp, i64, i64, vp, vp, i64, i64, i64, i32, i32, i32, vp]),
        "bsvd_tsmqr_fused": (i32, [vp, i64, i64, vp, vp, vp, i32, i64, i32, i32, i32, vp]),
    }
    for name, (res, args) in proto.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def lib():
    """Library handle for compute calls; fails loudly without a CUDA device."""
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device visible: the B200 engine has no CPU fallback")
    return load()


def check(status: int) -> None:
    """Raise the reference exception class matching a bsvd_status."""
    if status == BSVD_OK:
        return
    msg = load().bsvd_last_error().decode(errors="replace")
    if status == BSVD_E_SHAPE:
        raise ShapeError(msg)
    if status == BSVD_E_CONFIG:
        raise ConfigError(msg)
    if status == BSVD_E_VALIDATION:
        raise ValidationError(msg)
    if status == BSVD_E_CONVERGENCE:
        raise ConvergenceError(msg)
    raise DeviceError(f"bsvd status {status}: {msg}")


def make_config(cfg) -> BsvdConfig:
    return BsvdConfig(int(cfg.tilesize), int(cfg.colperblock or 0), int(cfg.splitk),
                      int(bool(cfg.fused)))
