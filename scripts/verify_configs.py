"""Run every BASELINE.json config once on the GPU: time + accuracy against the
known spectrum / host LAPACK (development + evidence script; results go to
profiles/).  Usage: python scripts/verify_configs.py [c1 c2 c3 c4 c5]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_06339_b200 as P

EPS = {torch.float64: 2.0 ** -52, torch.float32: 2.0 ** -23, torch.float16: 2.0 ** -10}


def errs(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return float(np.max(np.abs(got - want)) / want[0]), float(np.linalg.norm(got - want) / np.linalg.norm(want))


def timed(fn):
    """Wall time of one call after one warm-up call (workspace growth, module
    load and first-touch costs stay out of the number)."""
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t0


def run(name, a, ts, ref, dtype, tol_k=1.0):
    cfg = P.KernelConfig(tilesize=ts) if ts else None
    P.svdvals(a[:256, :256].contiguous(), cfg)              # warm the kernels
    vals, dt = timed(lambda: P.svdvals(a, cfg))
    n = a.shape[0]
    vals = vals.double().cpu().numpy()
    e_abs, e_nw = errs(vals, ref)
    bound = tol_k * (EPS[dtype] if dtype == torch.float16 else max(n, 16) * EPS[dtype])
    rec = {"config": name, "n": n, "dtype": str(dtype), "ts": ts or P.KernelConfig.for_size(n).tilesize,
           "seconds": dt, "tflops": 8 / 3 * n ** 3 / dt / 1e12, "max_abs_over_smax": e_abs,
           "normwise": e_nw, "bound": bound, "pass": e_abs <= bound and e_nw <= bound}
    print(json.dumps(rec), flush=True)
    return rec


def graded(n, cond, seed, dtype):
    g = torch.Generator(device="cuda").manual_seed(seed)
    sig = torch.logspace(0, -np.log10(cond), n, dtype=torch.float64, device="cuda")
    u, _ = torch.linalg.qr(torch.randn(n, n, generator=g, dtype=torch.float64, device="cuda"))
    v, _ = torch.linalg.qr(torch.randn(n, n, generator=g, dtype=torch.float64, device="cuda"))
    a = (u * sig) @ v.T
    return a.to(dtype), sig.cpu().numpy()


def main():
    which = sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"]
    out = []
    g = torch.Generator(device="cuda").manual_seed(0)
    if "c1" in which:
        a = torch.randn(1024, 1024, generator=g, device="cuda")
        ref = torch.linalg.svdvals(a.double()).cpu().numpy()
        out.append(run("C1 1024 fp32 ts32", a, 32, ref, torch.float32))
    if "c2" in which:
        a = torch.randn(8192, 8192, generator=g, device="cuda")
        ref = torch.linalg.svdvals(a.double()).cpu().numpy()
        out.append(run("C2 8192 fp32 default tiles", a, 0, ref, torch.float32))
    if "c3" in which:
        a, sig = graded(16384, 1e8, 3, torch.float64)
        out.append(run("C3 16384 fp64 graded cond 1e8 (vs known sigma)", a, 0, sig, torch.float64))
    if "c4" in which:
        a = torch.randn(8192, 8192, generator=g, device="cuda").half()
        ref = torch.linalg.svdvals(a.double()).cpu().numpy()
        out.append(run("C4 8192 fp16-storage", a, 0, ref, torch.float16))
    if "c5" in which:
        B, n = 4096, 512
        x = torch.randn(B, n, n, generator=g, device="cuda")
        P.svdvals_batched(x[:8])
        vals, dt = timed(lambda: P.svdvals_batched(x))
        idx = [0, 1, B // 2, B - 1]
        ref = torch.linalg.svdvals(x[idx].double()).cpu().numpy()
        got = vals[idx].double().cpu().numpy()
        e = max(errs(got[i], ref[i])[0] for i in range(len(idx)))
        rec = {"config": "C5 batch 4096 x 512^2 fp32 (1 GPU)", "seconds": dt,
               "tflops": B * 8 / 3 * n ** 3 / dt / 1e12, "max_abs_over_smax_sampled": e,
               "bound": n * EPS[torch.float32], "pass": e <= n * EPS[torch.float32]}
        print(json.dumps(rec), flush=True)
        out.append(rec)
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/verify_configs.json", "w"), indent=1)


if __name__ == "__main__":
    main()
