"""paper_2508_06339_b200 -- B200-native drop-in for the reference `bandsvd`
singular-value hot path (arXiv 2508.06339): dense -> band (tiled QR/LQ) ->
bidiagonal (bulge chase) -> values (Sturm bisection), all on sm_100a through
libbsvd.so (include/bsvd.h).  See DESIGN.md."""

from .api import (PHASE_KEYS, band_to_bidiagonal, banddiag, bidiagonal_values,
                  svdvals, svdvals_batched)
from .backend import B200Backend, LaunchStats, default_backend
from .config import KernelConfig
from .errors import (ConfigError, ConvergenceError, DegenerateInputError, DeviceError,
                     ExecutionModelError, FormatError, ShapeError, TileRangeError,
                     ValidationError)
from .matrix import DenseMatrix, pad_to_tiles, read_matrix, write_matrix
from .precision import FP16, FP32, FP64, Precision, by_name

__version__ = "0.1.0"

__all__ = [
    "svdvals", "svdvals_batched", "banddiag", "band_to_bidiagonal", "bidiagonal_values",
    "PHASE_KEYS", "B200Backend", "LaunchStats", "default_backend", "KernelConfig",
    "ConfigError", "ConvergenceError", "DegenerateInputError", "DeviceError",
    "ExecutionModelError", "FormatError", "ShapeError", "TileRangeError", "ValidationError",
    "DenseMatrix", "pad_to_tiles", "read_matrix", "write_matrix",
    "FP16", "FP32", "FP64", "Precision", "by_name", "__version__",
]
