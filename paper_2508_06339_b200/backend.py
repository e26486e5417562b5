"""B200Backend -- the reference's plugin object (execmodel.py:295-333 protocol:
``launch``, ``alloc_array``, ``free_array``, ``close``, ``stats``, context
manager), bound to one CUDA device.

Passed as ``svdvals(a, cfg, backend=B200Backend())`` it selects the GPU
pipeline (``stage1="tree"`` fast path or ``"faithful"`` reference-exact
stage 1).  Its ``launch`` is a kernel-level registry: the reference's tile
kernels (``geqrt_kernel``, ``tsqrt_kernel``, ``unmqr_kernel``,
``tsmqr_kernel``, kernels.py:205-421) run as their bit-faithful sm_100a
counterparts (``geqrt_splitk_kernel`` / ``tsqrt_splitk_kernel`` included,
kernels.py:233-361), so the reference's own driver (``bandsvd.banddiag`` /
``bandsvd.svdvals``) can execute stage 1 on the B200 unchanged.
"""
from __future__ import annotations

import contextlib
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigError, DeviceError


@dataclass
class LaunchStats:
    launches: int = 0
    barriers: int = 0
    shared_traffic: int = 0

    def delta_since(self, other: "LaunchStats") -> "LaunchStats":
        return LaunchStats(self.launches - other.launches, self.barriers - other.barriers,
                           self.shared_traffic - other.shared_traffic)

    def copy(self) -> "LaunchStats":
        return LaunchStats(self.launches, self.barriers, self.shared_traffic)


_DT_CODE = {np.dtype(np.float64): 1, np.dtype(np.float32): 2, np.dtype(np.float16): 3}


class B200Backend:
    """One CUDA device + stream + cached workspace."""

    checked = False

    def __init__(self, device: int | None = None, stage1: str = "tree", stream=None):
        import torch
        if stage1 not in ("tree", "faithful"):
            raise ConfigError(f"stage1 must be 'tree' or 'faithful', got {stage1!r}")
        if not torch.cuda.is_available():
            raise DeviceError("no CUDA device visible: the B200 engine has no CPU fallback")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.stage1 = stage1
        self.stream = stream
        self.stats = LaunchStats()
        self._tls = threading.local()   # workspace per host thread: concurrent calls never share it
        _lib.load()

    # ---- plumbing -------------------------------------------------------
    @property
    def stage1_algo(self) -> int:
        return _lib.STAGE1_FAITHFUL if self.stage1 == "faithful" else _lib.STAGE1_TREE

    def cuda_stream(self):
        import torch
        return self.stream if self.stream is not None else torch.cuda.current_stream(self.device)

    def stream_handle(self) -> int:
        return int(self.cuda_stream().cuda_stream)

    @contextlib.contextmanager
    def ordered(self, *tensors):
        """Order a library call on this backend's stream after the work the
        caller's current stream queued (inputs, outputs, workspace), and the
        caller's stream after the call; tensors touched on a foreign stream are
        marked with record_stream so the caching allocator does not hand
        their blocks out while the call may still use them."""
        import torch
        if self.stream is None:
            yield
            return
        cur = torch.cuda.current_stream(self.device)
        if self.stream == cur:
            yield
            return
        self.stream.wait_stream(cur)
        try:
            yield
        finally:
            for t in tensors:
                if t is not None and t.is_cuda:
                    t.record_stream(self.stream)
            cur.wait_stream(self.stream)

    def workspace(self, nbytes: int):
        """Cached device scratch of the calling host thread (grown on demand;
        stream-ordered reuse).  Per thread, so svdvals may be called
        concurrently on disjoint matrices."""
        import torch
        nbytes = max(int(nbytes), 256)
        ws = getattr(self._tls, "ws", None)
        if ws is None or ws.numel() < nbytes:
            self._tls.ws = None
            ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            self._tls.ws = ws
        return ws

    # ---- reference backend protocol ------------------------------------
    def alloc_array(self, size, dtype) -> np.ndarray:
        return np.zeros(size, dtype=dtype)

    def free_array(self, arr) -> None:
        pass

    def launch(self, kernel, spec, args):
        """Run a reference tile kernel (by name) as its faithful sm_100a twin.

        Views are staged to the device as column-major copies and written
        back, so any (possibly transposed) numpy view works; results are
        bit-identical to the reference interpreter's."""
        import torch
        name = getattr(kernel, "__name__", str(kernel))
        before = self.stats.copy()
        L = _lib.lib()
        st = self.stream_handle()

        def dev(arr):
            f = np.asfortranarray(arr)
            t = torch.from_numpy(np.ascontiguousarray(f.T)).to(self.device)
            return t, f.shape

        def back(t, arr):
            arr[...] = t.cpu().numpy().T

        if name in ("geqrt_kernel", "geqrt_splitk_kernel"):
            # geqrt_kernel(ctx, a, tau, ...) / geqrt_splitk_kernel(ctx, a, tau, nsplit, ...)
            a, tau = args[0], args[1]
            ts = a.shape[0]
            ta, _ = dev(a)
            tt = torch.from_numpy(np.array(tau)).to(self.device)
            if name == "geqrt_kernel":
                _lib.check(L.bsvd_geqrt(ta.data_ptr(), 1, ts, _DT_CODE[a.dtype], ts, tt.data_ptr(), st))
            else:
                _lib.check(L.bsvd_geqrt_splitk(ta.data_ptr(), 1, ts, _DT_CODE[a.dtype], ts, int(args[2]),
                                               tt.data_ptr(), st))
            back(ta, a)
            tau[...] = tt.cpu().numpy()
        elif name in ("tsqrt_kernel", "tsqrt_splitk_kernel"):
            # tsqrt_kernel(ctx, r, bs, taus, ...) / tsqrt_splitk_kernel(ctx, r, bs, taus, nsplit, ...)
            r, bs, taus = args[0], args[1], args[2]
            ts = r.shape[0]
            tr, _ = dev(r)
            tbs = [dev(b)[0] for b in bs]
            ttau = [torch.from_numpy(np.array(t)).to(self.device) for t in taus]
            pb = torch.tensor([t.data_ptr() for t in tbs], dtype=torch.int64, device=self.device)
            pt = torch.tensor([t.data_ptr() for t in ttau], dtype=torch.int64, device=self.device)
            if name == "tsqrt_kernel":
                _lib.check(L.bsvd_tsqrt_chain(tr.data_ptr(), 1, ts, pb.data_ptr(), pt.data_ptr(),
                                              len(bs), _DT_CODE[r.dtype], ts, st))
            else:
                _lib.check(L.bsvd_tsqrt_chain_splitk(tr.data_ptr(), 1, ts, pb.data_ptr(), pt.data_ptr(),
                                                     len(bs), _DT_CODE[r.dtype], ts, int(args[3]), st))
            back(tr, r)
            for t, b in zip(tbs, bs):
                back(t, b)
            for t, h in zip(ttau, taus):
                h[...] = t.cpu().numpy()
        elif name == "unmqr_kernel":
            panel, tau, x, cpb = args[0], args[1], args[2], args[3]
            ts = panel.shape[0]
            tp, _ = dev(panel)
            tx, _ = dev(x)
            tt = torch.from_numpy(np.array(tau)).to(self.device)
            _lib.check(L.bsvd_unmqr(tp.data_ptr(), 1, ts, tt.data_ptr(), tx.data_ptr(), 1, ts,
                                    x.shape[1], _DT_CODE[panel.dtype], ts, int(cpb), st))
            back(tx, x)
        elif name == "tsmqr_kernel":
            y, xs, vs, taus, cpb = args[0], args[1], args[2], args[3], args[4]
            ts = y.shape[0]
            ty, _ = dev(y)
            txs = [dev(x)[0] for x in xs]
            tvs = [dev(v)[0] for v in vs]
            ttau = [torch.from_numpy(np.array(t)).to(self.device) for t in taus]
            mk = lambda ts_: torch.tensor([t.data_ptr() for t in ts_], dtype=torch.int64, device=self.device)
            px, pv, pt = mk(txs), mk(tvs), mk(ttau)
            _lib.check(L.bsvd_tsmqr_fused(ty.data_ptr(), 1, ts, px.data_ptr(), pv.data_ptr(),
                                          pt.data_ptr(), len(xs), y.shape[1], _DT_CODE[y.dtype],
                                          ts, int(cpb), st))
            back(ty, y)
            for t, x in zip(txs, xs):
                back(t, x)
        else:
            raise ConfigError(f"B200Backend has no sm_100a kernel for {name!r}")
        self.cuda_stream().synchronize()
        self.stats.launches += 1
        return self.stats.delta_since(before)

    def close(self):
        self._tls = threading.local()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False


_default = {}


def default_backend() -> B200Backend:
    import torch
    dev = torch.cuda.current_device() if torch.cuda.is_available() else -1
    be = _default.get(dev)
    if be is None:
        be = B200Backend()
        _default[dev] = be
    return be

