"""Batch sharding host logic with world_size 2 on CPU (gloo): shard ranges,
per-rank compute, all-gather with uneven shards, rank ordering.  The per-rank
compute is the C oracle here (the GPU batched kernel is covered by
tests/test_gpu_parity.py); the collective path is the one NCCL runs."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, batch, n, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from oracle import oracle as O
    from paper_2508_06339_b200.distributed import shard_range, svdvals_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(7)
    a = rng.standard_normal((batch, n, n)).astype(np.float32)   # same global batch everywhere
    seen = []

    def compute(shard):
        seen.append(shard.shape[0])
        return torch.from_numpy(np.stack([O.svdvals(m, 4) for m in shard]) if len(shard)
                                else np.zeros((0, n), np.float32))

    vals = svdvals_sharded(a, _compute=compute)
    lo, hi = shard_range(batch, world, rank)
    # generator form: each rank builds only its own shard
    vals2 = svdvals_sharded(batch=batch, make_shard=lambda l, h: a[l:h], _compute=compute)
    np.save(os.path.join(out_dir, f"r{rank}.npy"), vals.numpy())
    np.save(os.path.join(out_dir, f"r{rank}_gen.npy"), vals2.numpy())
    np.save(os.path.join(out_dir, f"r{rank}_n.npy"), np.array([seen[0], hi - lo]))
    dist.destroy_process_group()


@pytest.mark.parametrize("batch", [5, 8])
def test_sharded_gather_world2(tmp_path, batch):
    from oracle import oracle as O
    n, world = 12, 2
    mp.spawn(_worker, args=(world, _free_port(), batch, n, str(tmp_path)), nprocs=world, join=True)
    a = np.random.default_rng(7).standard_normal((batch, n, n)).astype(np.float32)
    want = np.stack([O.svdvals(m, 4) for m in a])
    for r in range(world):
        got = np.load(tmp_path / f"r{r}.npy")
        assert np.array_equal(got, want)
        assert np.array_equal(np.load(tmp_path / f"r{r}_gen.npy"), want)
        seen, expect = np.load(tmp_path / f"r{r}_n.npy")
        assert seen == expect          # each rank computed only its own shard


def test_shard_range_partition():
    from paper_2508_06339_b200.distributed import shard_range
    for B in (0, 1, 7, 4096):
        for W in (1, 2, 4, 8):
            spans = [shard_range(B, W, r) for r in range(W)]
            assert spans[0][0] == 0 and spans[-1][1] == B
            assert all(spans[i][1] == spans[i + 1][0] for i in range(W - 1))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1
