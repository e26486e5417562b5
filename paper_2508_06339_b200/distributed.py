"""Batch sharding across GPUs.

A single matrix never leaves its GPU ("replicas only" for one matrix).  A batch
of B independent matrices is split into contiguous shards, rank r of W taking
matrices [r*B//W, (r+1)*B//W); each rank runs the batched sm_100a pipeline on
its shard and ONE collective -- an all-gather of the values over NCCL
(NVLink/NVSwitch) -- assembles the [B, n] result on every rank.  Inputs never
cross the interconnect: callers hand every rank either the global batch (it
slices its own shard) or a shard generator.

The reference farms matrices over worker processes with a ProcessPoolExecutor
(bench.py:161-189); this is the multi-GPU analogue.
"""
from __future__ import annotations

from typing import Callable

import numpy as np


def shard_range(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced shard [lo, hi) of `batch` items for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    return batch * rank // world, batch * (rank + 1) // world


def gather_values(local, batch: int, n: int, group=None):
    """All-gather per-rank value blocks [b_r, n] into [batch, n] (rank order).

    Shards may differ in size by one; blocks are padded to the largest shard
    for the collective and trimmed afterwards.  Works for any backend
    (NCCL on the GPU path, gloo in the CPU tests)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    sizes = [shard_range(batch, world, r) for r in range(world)]
    maxb = max(hi - lo for lo, hi in sizes)
    pad = torch.zeros((maxb, n), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return torch.cat([o[: hi - lo] for o, (lo, hi) in zip(outs, sizes)], dim=0)


def svdvals_sharded(a=None, cfg=None, backend=None, group=None, *, batch: int | None = None,
                    make_shard: Callable[[int, int], object] | None = None,
                    _compute: Callable | None = None):
    """Singular values of a batch of independent matrices sharded over the
    ranks of `group` (torch.distributed, one process per GPU).

    Pass either `a` ([B, n, n], every rank the same global batch; each rank
    only touches its shard) or `batch` + `make_shard(lo, hi)` returning the
    rank's own [hi-lo, n, n] shard.  Returns the gathered [B, n] values (a
    device tensor on the GPU path).  `_compute` replaces the GPU batched call
    (used by the gloo CPU tests)."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if a is not None:
        B = int(a.shape[0])
        lo, hi = shard_range(B, world, rank)
        shard = a[lo:hi]
    else:
        if batch is None or make_shard is None:
            raise ValueError("pass the global batch `a`, or `batch` and `make_shard`")
        B = int(batch)
        lo, hi = shard_range(B, world, rank)
        shard = make_shard(lo, hi)
    n = int(shard.shape[-1])
    if _compute is None:
        from .api import svdvals_batched
        if hi > lo:
            local = svdvals_batched(shard if isinstance(shard, torch.Tensor) else np.asarray(shard),
                                    cfg, backend)
            local = local if isinstance(local, torch.Tensor) else torch.from_numpy(local)
        else:
            # same dtype as the other ranks' blocks (FP64 -> float64, else
            # float32): all_gather needs equal element sizes on every rank
            sdt = getattr(shard, "dtype", None)
            f64 = sdt in (torch.float64, np.float64, np.dtype(np.float64))
            local = torch.zeros((0, n), dtype=torch.float64 if f64 else torch.float32)
        if dist.get_backend(group) == "nccl":
            local = local.cuda()
    else:
        local = _compute(shard)
    return gather_values(local, B, n, group)
