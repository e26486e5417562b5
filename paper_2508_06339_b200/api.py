"""Public entry points -- drop-ins for the reference hot path.

* ``svdvals(a, cfg=None, backend=None, timers=None)``  secondstage.py:510-542
* ``svdvals_batched(a, cfg=None, backend=None, timers=None)``  batch of
  independent matrices (the reference farms them over processes,
  bench.py:161-189; here one call covers the batch)
* ``banddiag(a, cfg=None, backend=None)``               bandreduce.py:91-120
* ``band_to_bidiagonal(band, bandwidth, backend=None)`` secondstage.py:452-470
* ``bidiagonal_values(d, e, backend=None)``             secondstage.py:473-507

Everything runs on the GPU through libbsvd.so (include/bsvd.h); there is no
CPU fallback.  Host inputs (numpy / DenseMatrix) are copied to the device
column-major exactly like ``DenseMatrix.from_array`` lays them out, results
come back as numpy arrays in the compute dtype (FP16 -> float32), like the
reference.  torch CUDA tensors are consumed in place by ``svdvals`` (a row-major tensor
is read as its transpose: sigma(A) = sigma(A^T)); the stage entry points copy
a row-major tensor to column-major first.  Device results stay on the device.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .backend import B200Backend, default_backend
from .config import KernelConfig
from .errors import ConfigError, ShapeError
from .precision import FP16, FP32, FP64, from_storage_dtype

PHASE_KEYS = ("panel", "trailing", "bidiagonal", "diagonal")


def _backend(backend) -> B200Backend:
    if backend is None:
        return default_backend()
    if isinstance(backend, B200Backend):
        return backend
    raise ConfigError(
        f"backend {type(backend).__name__} is not a B200Backend; this engine executes on the "
        "GPU only (pass backend=None or a B200Backend)")


def _torch():
    import torch
    return torch


def _torch_prec(t):
    torch = _torch()
    return {torch.float64: FP64, torch.float32: FP32, torch.float16: FP16}.get(t.dtype)


def _as_device_matrix(a, be: B200Backend, transpose_ok: bool = True):
    """-> (tensor on device, precision, n, lda, is_host_input, n_out).

    The tensor's memory holds the matrix column-major with leading dim lda.
    With ``transpose_ok`` (svdvals: sigma(A) = sigma(A^T)) a row-major torch
    tensor is read in place as the column-major A^T; the stage entry points
    (whose outputs are not transpose-invariant) get a real column-major copy.
    ``n_out`` is the number of values the reference returns (``orig_n`` of a
    padded DenseMatrix, secondstage.py:523,542)."""
    torch = _torch()
    if isinstance(a, torch.Tensor):
        if a.ndim != 2:
            raise ShapeError(f"expected a 2-D array, got ndim={a.ndim}")
        prec = _torch_prec(a)
        if prec is None:
            a = a.to(torch.float64)
            prec = FP64
        if a.shape[0] != a.shape[1]:
            raise ShapeError(f"matrix must be square, got {a.shape[0]}x{a.shape[1]}")
        host = not a.is_cuda
        t = a.to(be.device) if host else a
        n = t.shape[0]
        if t.stride(0) == 1 and t.stride(1) >= n:
            return t, prec, n, t.stride(1), host, n       # column-major A
        if transpose_ok and t.stride(1) == 1 and t.stride(0) >= n:
            return t, prec, n, t.stride(0), host, n       # read as A^T
        t = t.t().contiguous()                            # memory = column-major A
        return t, prec, n, n, host, n
    # numpy / DenseMatrix (ours or the reference's): column-major storage copy
    if hasattr(a, "array") and hasattr(a, "precision") and not isinstance(a, np.ndarray):
        arr = np.asarray(a.array)
        prec = from_storage_dtype(arr.dtype)
        n_orig = getattr(a, "orig_n", None)
    else:
        arr = np.asarray(a)
        if arr.ndim != 2:
            raise ShapeError(f"expected a 2-D array, got ndim={arr.ndim}")
        prec = from_storage_dtype(arr.dtype) if arr.dtype in (
            np.dtype(np.float64), np.dtype(np.float32), np.dtype(np.float16)) else FP64
        n_orig = None
    if arr.shape[0] != arr.shape[1]:
        raise ShapeError(f"matrix must be square, got {arr.shape[0]}x{arr.shape[1]}")
    if arr.shape[0] < 1:
        raise ShapeError("matrix must have size >= 1")
    f = np.asfortranarray(arr, dtype=prec.storage_dtype)
    t = torch.from_numpy(f.T).to(be.device, non_blocking=False)   # memory = column-major A
    n_out = arr.shape[0] if n_orig is None else max(1, min(int(n_orig), arr.shape[0]))
    return t, prec, arr.shape[0], arr.shape[0], True, n_out


def _out_torch_dtype(prec):
    torch = _torch()
    return torch.float64 if prec is FP64 else torch.float32


def _add_timers(timers, tm):
    if timers is not None:
        timers["panel"] += tm.panel_s
        timers["trailing"] += tm.trailing_s
        timers["bidiagonal"] += tm.bidiagonal_s
        timers["diagonal"] += tm.diagonal_s


def _prep_timers(timers):
    if timers is None:
        return None
    for k in PHASE_KEYS:
        timers.setdefault(k, 0.0)
    return _lib.BsvdTimers()


def svdvals(a, cfg: KernelConfig | None = None, backend=None, timers=None):
    """All singular values of a square matrix, descending, in its compute
    precision (secondstage.py:510-542).  ShapeError for non-square / empty,
    ValidationError for NaN/Inf (checked before any stage runs)."""
    torch = _torch()
    be = _backend(backend)
    L = _lib.lib()
    t, prec, n, lda, host, n_out = _as_device_matrix(a, be)
    if n < 1:
        raise ShapeError("matrix must have size >= 1")
    cfg = cfg if cfg is not None else KernelConfig.for_size(n)
    ccfg = _lib.make_config(cfg)
    opt = _lib.BsvdOptions()
    L.bsvd_default_options(ctypes.byref(opt))
    opt.stage1_algo = be.stage1_algo
    nbytes = L.bsvd_workspace_bytes(prec.code, n, 1, ctypes.byref(ccfg))
    ws = be.workspace(nbytes)
    out = torch.empty(n, dtype=_out_torch_dtype(prec), device=be.device)
    tm = _prep_timers(timers)
    with torch.cuda.device(be.device), be.ordered(t, out, ws):
        _lib.check(L.bsvd_svdvals_ex(t.data_ptr(), prec.code, n, lda, ctypes.byref(ccfg),
                                     ctypes.byref(opt), out.data_ptr(), ws.data_ptr(), ws.numel(),
                                     be.stream_handle(), ctypes.byref(tm) if tm is not None else None))
    _add_timers(timers, tm)
    be.stats.launches += 1
    if n_out < n:
        out = out[:n_out]
    if host:
        return out.cpu().numpy()
    return out


def svdvals_batched(a, cfg: KernelConfig | None = None, backend=None, timers=None):
    """Singular values of a batch [B, n, n] of independent square matrices
    -> [B, n] (descending per row).  Each matrix is read as its transpose
    when the batch is row-major (values are transpose-invariant)."""
    torch = _torch()
    be = _backend(backend)
    L = _lib.lib()
    host = not (isinstance(a, torch.Tensor) and a.is_cuda)
    if not isinstance(a, torch.Tensor):
        arr = np.asarray(a)
        if arr.dtype not in (np.float64, np.float32, np.float16):
            arr = arr.astype(np.float64)
        a = torch.from_numpy(np.ascontiguousarray(arr))
    if a.ndim != 3 or a.shape[1] != a.shape[2]:
        raise ShapeError(f"expected a [batch, n, n] array, got shape {tuple(a.shape)}")
    prec = _torch_prec(a)
    if prec is None:
        a, prec = a.to(torch.float64), FP64
    t = a.to(be.device).contiguous()
    B, n = t.shape[0], t.shape[1]
    if n < 1 or B < 1:
        raise ShapeError("batch and matrix size must be >= 1")
    cfg = cfg if cfg is not None else KernelConfig.for_size(n)
    ccfg = _lib.make_config(cfg)
    nbytes = L.bsvd_workspace_bytes(prec.code, n, B, ctypes.byref(ccfg))
    ws = be.workspace(nbytes)
    out = torch.empty((B, n), dtype=_out_torch_dtype(prec), device=be.device)
    tm = _prep_timers(timers)
    with torch.cuda.device(be.device), be.ordered(t, out, ws):
        _lib.check(L.bsvd_svdvals_batched(t.data_ptr(), prec.code, n, n, n * n, B,
                                          ctypes.byref(ccfg), out.data_ptr(), ws.data_ptr(),
                                          ws.numel(), be.stream_handle(),
                                          ctypes.byref(tm) if tm is not None else None))
    _add_timers(timers, tm)
    be.stats.launches += 1
    return out.cpu().numpy() if host else out


def banddiag(a, cfg: KernelConfig | None = None, backend=None):
    """Stage 1 only: reduce a square matrix (zero-padded to a multiple of
    cfg.tilesize) to upper-band form, band width = tilesize, exact zeros
    outside the band (bandreduce.py:91-120).  Returns the padded band as a
    column-major (Fortran-order) numpy array in the storage dtype, or (device
    input) a device tensor whose value is the band, stored column-major."""
    torch = _torch()
    be = _backend(backend)
    L = _lib.lib()
    t, prec, n, lda, host, _ = _as_device_matrix(a, be, transpose_ok=False)
    cfg = cfg if cfg is not None else KernelConfig.for_size(n)
    ts = cfg.tilesize
    N = max(1, -(-n // ts))
    npad = N * ts
    # padded column-major working copy (ld = npad)
    work = torch.zeros((npad, npad), dtype=t.dtype, device=be.device)   # row-major storage of A^T
    # src[j, i] = M[i, j]: row-major view of M's column-major memory
    work[:n, :n].copy_(torch.as_strided(t, (n, n), (lda, 1), t.storage_offset()))
    ccfg = _lib.make_config(cfg)
    opt = _lib.BsvdOptions()
    L.bsvd_default_options(ctypes.byref(opt))
    opt.stage1_algo = be.stage1_algo
    nbytes = L.bsvd_workspace_bytes(prec.code, npad, 1, ctypes.byref(ccfg))
    ws = be.workspace(nbytes)
    with torch.cuda.device(be.device), be.ordered(work, ws):
        _lib.check(L.bsvd_banddiag(work.data_ptr(), prec.code, npad, ctypes.byref(ccfg),
                                   ctypes.byref(opt), ws.data_ptr(), ws.numel(), be.stream_handle()))
    if host:
        return work.cpu().numpy().T          # Fortran-order view: band of A
    return work.t()                          # the band itself (column-major strides)


def band_to_bidiagonal(band, bandwidth: int, backend=None):
    """Stage 2 only: upper band (square, band width ``bandwidth``) -> float64
    (d, e) by the pipelined Householder bulge chase (secondstage.py:452-470
    computes the same bidiagonal's singular values by Givens rotations)."""
    torch = _torch()
    be = _backend(backend)
    L = _lib.lib()
    t, prec, n, lda, host, _ = _as_device_matrix(band, be, transpose_ok=False)
    t = torch.as_strided(t, (n, n), (lda, 1), t.storage_offset()).contiguous()
    d = torch.empty(n, dtype=torch.float64, device=be.device)
    e = torch.empty(max(n - 1, 1), dtype=torch.float64, device=be.device)
    if not 1 <= bandwidth <= 128:
        raise ConfigError(f"band width must lie in [1, 128], got {bandwidth}")
    ws = be.workspace(L.bsvd_band_workspace_bytes(n, int(bandwidth)))
    with torch.cuda.device(be.device), be.ordered(t, d, e, ws):
        _lib.check(L.bsvd_band_to_bidiagonal(t.data_ptr(), prec.code, n, int(bandwidth),
                                             d.data_ptr(), e.data_ptr(), ws.data_ptr(), ws.numel(),
                                             be.stream_handle()))
    e = e[: n - 1]
    if host:
        return d.cpu().numpy(), e.cpu().numpy()
    return d, e


def bidiagonal_values(d, e, backend=None):
    """Stage 3 only: all singular values (descending, float64) of the upper
    bidiagonal (d, e) by GPU Sturm bisection (secondstage.py:473-507)."""
    torch = _torch()
    be = _backend(backend)
    L = _lib.lib()
    host = not (isinstance(d, torch.Tensor) and d.is_cuda)
    td = torch.as_tensor(np.asarray(d) if host else d, dtype=torch.float64).to(be.device).contiguous()
    n = td.numel()
    if n < 1:
        raise ShapeError("bidiagonal matrix must have size >= 1")
    te = torch.as_tensor(np.asarray(e) if host else e, dtype=torch.float64).to(be.device).contiguous()
    if te.numel() != n - 1:
        raise ShapeError(f"superdiagonal has {te.numel()} entries, expected {n - 1}")
    if te.numel() == 0:
        te = torch.zeros(1, dtype=torch.float64, device=be.device)
    out = torch.empty(n, dtype=torch.float64, device=be.device)
    with torch.cuda.device(be.device), be.ordered(td, te, out):
        _lib.check(L.bsvd_bidiagonal_values(td.data_ptr(), te.data_ptr(), n, out.data_ptr(),
                                            be.stream_handle()))
    return out.cpu().numpy() if host else out
