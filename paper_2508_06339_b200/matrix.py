"""Column-major matrix storage and the BSVD file format (reference
matrix.py:22-90, :163-181, :218-249).

The engine itself consumes numpy arrays, ``DenseMatrix`` objects (this
module's or the reference's -- anything exposing ``.array`` and
``.precision``) and torch tensors; ``DenseMatrix`` is kept so reference
call sites (``svdvals(DenseMatrix.from_array(a))``) port unchanged."""
from __future__ import annotations

import struct

import numpy as np

from .errors import FormatError, ShapeError
from .precision import FP64, Precision, from_storage_dtype

_MAGIC = b"BSVD"
_FORMAT_VERSION = 1
_DTYPE_CODES = {1: np.dtype("<f8"), 2: np.dtype("<f4"), 3: np.dtype("<f2")}
_CODE_FOR_KIND = {np.dtype(np.float64): 1, np.dtype(np.float32): 2, np.dtype(np.float16): 3}


class DenseMatrix:
    """rows x cols elements in one column-major buffer; (r, c) at c*rows + r."""

    __slots__ = ("rows", "cols", "orig_n", "data", "precision")

    def __init__(self, data: np.ndarray, rows: int, cols: int, orig_n: int | None = None,
                 precision: Precision | None = None):
        if data.ndim != 1:
            raise ShapeError("DenseMatrix data must be a 1-D buffer")
        if data.size != rows * cols:
            raise ShapeError(f"buffer holds {data.size} elements, need {rows}x{cols}")
        self.data = data
        self.rows = rows
        self.cols = cols
        self.orig_n = rows if orig_n is None else orig_n
        self.precision = precision if precision is not None else from_storage_dtype(data.dtype)
        if self.precision.storage_dtype != data.dtype:
            raise ShapeError(f"buffer dtype {data.dtype} does not match precision {self.precision.name}")

    @classmethod
    def zeros(cls, rows: int, cols: int, precision: Precision = FP64) -> "DenseMatrix":
        return cls(np.zeros(rows * cols, dtype=precision.storage_dtype), rows, cols, precision=precision)

    @classmethod
    def from_array(cls, arr, precision: Precision | None = None) -> "DenseMatrix":
        """Copy a 2-D array into column-major storage (rounding if needed)."""
        arr = np.asarray(arr)
        if arr.ndim != 2:
            raise ShapeError(f"expected a 2-D array, got ndim={arr.ndim}")
        if precision is None:
            precision = from_storage_dtype(arr.dtype) if arr.dtype in (
                np.dtype(np.float64), np.dtype(np.float32), np.dtype(np.float16)) else FP64
        rows, cols = arr.shape
        data = np.asfortranarray(arr, dtype=precision.storage_dtype).reshape(-1, order="F")
        return cls(data.copy(), rows, cols, precision=precision)

    @property
    def array(self) -> np.ndarray:
        return self.data.reshape((self.rows, self.cols), order="F")

    def copy(self) -> "DenseMatrix":
        return DenseMatrix(self.data.copy(), self.rows, self.cols, self.orig_n, self.precision)

    def __repr__(self):
        return f"DenseMatrix({self.rows}x{self.cols}, {self.precision.name}, orig_n={self.orig_n})"


def pad_to_tiles(m: DenseMatrix, ts: int) -> DenseMatrix:
    """Zero-pad a square matrix to the next multiple of ts (matrix.py:163-181)."""
    if m.rows != m.cols:
        raise ShapeError(f"cannot pad a non-square matrix ({m.rows}x{m.cols})")
    if ts < 1:
        raise ShapeError(f"tilesize must be positive, got {ts}")
    if m.rows % ts == 0 and m.rows > 0:
        return m
    nbtiles = max(1, -(-m.rows // ts))
    n = nbtiles * ts
    out = DenseMatrix.zeros(n, n, m.precision)
    out.orig_n = m.orig_n
    out.array[:m.rows, :m.cols] = m.array
    return out


def write_matrix(m: DenseMatrix, path) -> None:
    """magic 'BSVD' | version u32 | dtype code u32 | rows u64 | cols u64 |
    column-major little-endian payload (matrix.py:218-227)."""
    code = _CODE_FOR_KIND[m.data.dtype]
    le = _DTYPE_CODES[code]
    with open(path, "wb") as f:
        f.write(_MAGIC)
        f.write(struct.pack("<IIQQ", _FORMAT_VERSION, code, m.rows, m.cols))
        f.write(np.ascontiguousarray(m.data, dtype=le).tobytes())


def _read_header(path):
    """(dtype, rows, cols, payload bytes) with the reference's format errors
    (matrix.py:230-249), reading only the 28-byte header."""
    import os
    size = os.path.getsize(path)
    with open(path, "rb") as f:
        head = f.read(28)
    if len(head) < 4 or head[:4] != _MAGIC:
        raise FormatError(f"bad magic {head[:4]!r}, expected {_MAGIC!r}")
    if len(head) < 28:
        raise FormatError("truncated header")
    version, code, rows, cols = struct.unpack("<IIQQ", head[4:28])
    if version != _FORMAT_VERSION:
        raise FormatError(f"unknown format version {version}")
    if code not in _DTYPE_CODES:
        raise FormatError(f"unknown dtype code {code}")
    dtype = _DTYPE_CODES[code]
    expected = rows * cols * dtype.itemsize
    payload = size - 28
    if payload < expected:
        raise FormatError(f"truncated payload: {payload} bytes, expected {expected}")
    if payload > expected:
        raise FormatError(f"payload has {payload - expected} trailing bytes")
    return dtype, int(rows), int(cols)


def read_matrix_device(path, device=None, chunk_bytes: int = 64 << 20):
    """BSVD file -> device tensor without a host copy of the whole payload:
    the payload is memory-mapped and streamed through two pinned staging
    buffers (the read of chunk i+1 overlaps the H2D copy of chunk i on a side
    stream).  Returns (tensor [rows, cols] whose memory is the column-major
    matrix -- i.e. the transposed view of the payload, as ``svdvals`` and
    ``banddiag`` consume it --, precision).  SURVEY.md 8(f) row 2."""
    import torch
    dtype, rows, cols = _read_header(path)
    native = dtype.newbyteorder("=")
    mm = np.memmap(path, dtype=dtype, mode="r", offset=28, shape=(rows * cols,))
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    tdt = {1: torch.float64, 2: torch.float32, 3: torch.float16}[
        {np.dtype("<f8"): 1, np.dtype("<f4"): 2, np.dtype("<f2"): 3}[np.dtype(dtype)]]
    out = torch.empty(rows * cols, dtype=tdt, device=dev)
    per = max(1, chunk_bytes // dtype.itemsize)
    bufs = [torch.empty(min(per, rows * cols), dtype=tdt, pin_memory=True) for _ in range(2)]
    events = [None, None]
    stream = torch.cuda.Stream(device=dev)
    for i, lo in enumerate(range(0, rows * cols, per)):
        hi = min(rows * cols, lo + per)
        b = i & 1
        if events[b] is not None:
            events[b].synchronize()          # the copy out of this buffer is done
        bufs[b].numpy()[: hi - lo] = mm[lo:hi].astype(native, copy=False)
        with torch.cuda.stream(stream):
            out[lo:hi].copy_(bufs[b][: hi - lo], non_blocking=True)
            events[b] = torch.cuda.Event()
            events[b].record(stream)
    torch.cuda.current_stream(dev).wait_stream(stream)
    out.record_stream(stream)
    del mm
    return out.view(cols, rows).t(), from_storage_dtype(np.dtype(native))


def read_matrix(path) -> DenseMatrix:
    """Inverse of write_matrix with the reference's format errors (:230-249)."""
    with open(path, "rb") as f:
        raw = f.read()
    if len(raw) < 4 or raw[:4] != _MAGIC:
        raise FormatError(f"bad magic {raw[:4]!r}, expected {_MAGIC!r}")
    if len(raw) < 28:
        raise FormatError("truncated header")
    version, code, rows, cols = struct.unpack("<IIQQ", raw[4:28])
    if version != _FORMAT_VERSION:
        raise FormatError(f"unknown format version {version}")
    if code not in _DTYPE_CODES:
        raise FormatError(f"unknown dtype code {code}")
    dtype = _DTYPE_CODES[code]
    expected = rows * cols * dtype.itemsize
    payload = raw[28:]
    if len(payload) < expected:
        raise FormatError(f"truncated payload: {len(payload)} bytes, expected {expected}")
    if len(payload) > expected:
        raise FormatError(f"payload has {len(payload) - expected} trailing bytes")
    data = np.frombuffer(payload, dtype=dtype).astype(dtype.newbyteorder("="), copy=True)
    return DenseMatrix(data, int(rows), int(cols))
