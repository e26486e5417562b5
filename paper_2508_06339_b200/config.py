"""KernelConfig -- the reference's tunables with identical validation
(kernels.py:32-64).  ``tilesize`` is the tile edge AND the band width of the
stage-1 output (bandreduce.py:110).  On the B200 engine ``colperblock`` and
``splitk`` are accepted and validated exactly like the reference; the fast
stage-1 path picks its own column blocking (they may only change rounding
order), the faithful path honours ``colperblock``."""
from __future__ import annotations

from dataclasses import dataclass

from .errors import ConfigError


@dataclass(frozen=True)
class KernelConfig:
    tilesize: int = 32
    colperblock: int | None = None
    splitk: int = 1
    fused: bool = True

    def __post_init__(self):
        ts = self.tilesize
        if not isinstance(ts, int) or not 4 <= ts <= 128:
            raise ConfigError(f"tilesize must be an integer in [4, 128], got {ts}")
        if self.colperblock is None:
            object.__setattr__(self, "colperblock", ts)
        cpb = self.colperblock
        if not isinstance(cpb, int) or not 1 <= cpb <= ts or ts % cpb:
            raise ConfigError(f"colperblock must divide tilesize and lie in [1, {ts}], got {cpb}")
        kmax = min(ts, 1024 // ts)
        if not isinstance(self.splitk, int) or not 1 <= self.splitk <= kmax:
            raise ConfigError(
                f"splitk must lie in [1, min(TILESIZE, 1024/TILESIZE)] = [1, {kmax}], "
                f"got {self.splitk}")

    @staticmethod
    def for_size(n: int) -> "KernelConfig":
        """kernels.py:57-64: ts = 4, doubled while ts < 128 and 8*ts < n."""
        ts = 4
        while ts < 128 and ts * 8 < n:
            ts *= 2
        return KernelConfig(tilesize=ts)
