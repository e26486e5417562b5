"""Benchmark: singular values of a dense matrix on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload single|batch] [--n 8192] [--dtype fp32]

A "step" is one pass of the hot path (secondstage.py:510-542 svdvals: pad ->
tiled QR/LQ band reduction -> bulge chase -> Sturm bisection) over one batch
of synthetic input already resident in HBM.  Default workload = BASELINE.json
configs[1]: one 8192 x 8192 FP32 N(0,1) matrix per GPU, default tiles
(KernelConfig.for_size(8192) -> ts = 128).  Throughput is TFLOP/s on the
reference's 8/3 n^3 flop model (whole job = all ranks), higher is better.
For N > 1 every rank reduces its own matrix ("a single matrix stays on one
GPU") and the values are gathered to all ranks with NCCL inside the step
(weak scaling).  `--workload batch` runs configs[4] instead: a batch of
independent 512 x 512 FP32 matrices (ts = 64) sharded across the ranks.

`--gpus N > 1` defaults to the sharded batch (configs[4]) through
`distributed.svdvals_sharded` (one NCCL all-gather of the values per step).

`--impl reference` times the reference's CPU path -- the bit-exact C port of
the reference (oracle/, "kind": "port"; the reference is Python+numba with no
compiled core to link) -- on the host's cores, rank 0 only.  An 8192^2 run of
the port takes minutes, so each step times a bounded 2048^2 sample (ts = 128);
the reported value is the c*n^3 fit of the samples (1024, 2048, 4096)
extrapolated to the workload's n, marked "extrapolated": true.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
CPU_SAMPLE_N = 2048
CPU_FIT_NS = (1024, 2048, 4096)


def flop_model(n: int) -> float:
    """8/3 n^3 (BASELINE.json metric)."""
    return 8.0 / 3.0 * float(n) ** 3


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6542.1), d.get("sm_max_mhz", 1965.0), "measured (MEASURED_PEAKS.json)"
    return 6650.0, 1965.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self):
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        load = [s for s in sm if s > 500] or sm
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _port_seconds(n, threads):
    """One svdvals of an n x n FP32 N(0,1) matrix (ts = 128) on the C port."""
    import numpy as np
    from oracle import oracle as O
    O.lib()
    O.set_num_threads(threads)
    a = np.random.default_rng(0xBE7C).standard_normal((n, n)).astype(np.float32)
    t0 = time.perf_counter()
    O.svdvals(a, 128)
    return time.perf_counter() - t0


def cpu_fit(samples, n_target):
    """c from t = c n^3 (least squares in log space) -> (seconds at n_target, c)."""
    import math
    logc = [math.log(t / float(n) ** 3) for n, t in samples]
    c = math.exp(sum(logc) / len(logc))
    return c * float(n_target) ** 3, c


def cpu_baseline_fit(n_target, threads=None, extra=()):
    """The reference's CPU path (C port, all host threads) at 1024/2048/4096,
    fitted c*n^3 and extrapolated to n_target; returns the cpu_baseline dict."""
    th = threads or os.cpu_count() or 1
    pts = [(n, _port_seconds(n, th)) for n in CPU_FIT_NS] + list(extra)
    t_target, c = cpu_fit(pts, n_target)
    return {"value": flop_model(n_target) / t_target / 1e12, "unit": "TFLOP/s", "cores": th, "kind": "port",
            "extrapolated": True, "seconds_at_n": t_target, "n": n_target,
            "fit": {"model": "t = c n^3", "c": c, "points_s": {str(n): t for n, t in pts}},
            "cpu_model": cpu_model(),
            "sample": (f"reference C port (oracle/bsvd_oracle.c, bit-exact to bandsvd) svdvals of "
                       f"{'/'.join(str(n) for n in CPU_FIT_NS)}^2 FP32 N(0,1) matrices, ts=128, {th} OpenMP "
                       f"threads, fitted t = c n^3 and extrapolated to n = {n_target}")}


def cpu_batch_sample(n, cnt, th):
    """Seconds for `cnt` independent n^2 FP32 matrices (ts = for_size(n)) on the
    C port, one after another with all threads each."""
    import numpy as np
    from oracle import oracle as O
    O.lib()
    O.set_num_threads(th)
    mats = np.random.default_rng(0xC5).standard_normal((cnt, n, n)).astype(np.float32)
    ts = O.default_tilesize(n)
    t0 = time.perf_counter()
    for i in range(cnt):
        O.svdvals(mats[i], ts)
    return time.perf_counter() - t0


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    th = os.cpu_count() or 1
    batch = workload_of(args) == "batch"
    if batch:
        # configs[4]: independent 512^2 FP32 matrices (ts = 64); each step runs a
        # bounded sample of 16 of them on the port (all threads per matrix)
        n, cnt = args.n or 512, 16
        one_step = lambda: cpu_batch_sample(n, cnt, th)
        for _ in range(args.warmup):
            one_step()
        step_s = statistics.median([one_step() for _ in range(args.steps)])
        v = cnt * flop_model(n) / step_s / 1e12
        base = {"value": v, "unit": "TFLOP/s", "cores": th, "kind": "port", "extrapolated": False,
                "cpu_model": cpu_model(),
                "sample": f"reference C port svdvals of {cnt} independent {n}^2 FP32 matrices per step, ts=64, "
                          f"{th} OpenMP threads per matrix"}
        cfg = {"workload": f"configs[4] sample: {cnt} of the 4096 independent {n}^2 FP32 matrices per step",
               "n": n, "tilesize": 64}
        sample_v = v
    else:
        n_target = args.n or 8192
        for _ in range(args.warmup):
            _port_seconds(CPU_SAMPLE_N, th)
        step_s = statistics.median([_port_seconds(CPU_SAMPLE_N, th) for _ in range(args.steps)])
        base = cpu_baseline_fit(n_target, th, extra=[(CPU_SAMPLE_N, step_s)])
        v = base["value"]
        cfg = {"workload": f"configs[1] (n = {n_target}, FP32, ts = 128) extrapolated from bounded CPU "
                           f"samples: each step one {CPU_SAMPLE_N}^2 svdvals, plus one 1024^2 and one "
                           "4096^2 for the c*n^3 fit",
               "n": n_target, "tilesize": 128}
        sample_v = flop_model(CPU_SAMPLE_N) / step_s / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (N(0,1), seeded)", "config": cfg, "sample_value": sample_v,
        "cpu_baseline": dict(base, value=v),
        "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_of(args):
    return args.workload or ("batch" if args.gpus > 1 or int(os.environ.get("WORLD_SIZE", 1)) > 1 else "single")


def run_b200(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2508_06339_b200 as P

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    be = P.B200Backend(device=local)
    L = P._lib.lib()
    dtype = {"fp32": torch.float32, "fp64": torch.float64, "fp16": torch.float16}[args.dtype]
    gen = torch.Generator(device=dev)
    gen.manual_seed(1000 + rank)

    from paper_2508_06339_b200 import distributed as D
    wl = workload_of(args)
    if wl == "single":
        n = args.n or 8192
        cfg = P.KernelConfig.for_size(n) if not args.ts else P.KernelConfig(tilesize=args.ts)
        x = torch.randn((n, n), generator=gen, device=dev, dtype=torch.float32).to(dtype)
        units, total_units = 1, world
        call = lambda inp, timers=None: P.svdvals(inp, cfg, be, timers)
        workload = (f"configs[1]: one {n}x{n} {args.dtype.upper()} N(0,1) matrix per GPU, svdvals "
                    f"(all singular values), default tiles ts={cfg.tilesize}")
        parallelism = (f"replicas x{world} (a single matrix stays on one GPU; values all-gathered over NCCL)"
                       if world > 1 else "1 GPU")

        def step(inp, timers=None):
            vals = call(inp, timers)
            if world > 1:
                vt = vals if isinstance(vals, torch.Tensor) else torch.from_numpy(vals).to(dev)
                out = [torch.empty_like(vt) for _ in range(world)]
                dist.all_gather(out, vt.contiguous())
                return out
            return vals
    else:
        n = args.n or 512
        total_units = args.batch or 4096
        lo, hi = D.shard_range(total_units, world, rank)
        units = hi - lo
        cfg = P.KernelConfig.for_size(n) if not args.ts else P.KernelConfig(tilesize=args.ts)
        # each rank generates its own shard (inputs never cross NVLink)
        x = torch.randn((units, n, n), generator=gen, device=dev, dtype=torch.float32).to(dtype)
        call = lambda inp, timers=None: P.svdvals_batched(inp, cfg, be, timers)
        workload = (f"configs[4]: batch of {total_units} independent {n}x{n} {args.dtype.upper()} matrices "
                    f"sharded {units} per GPU, ts={cfg.tilesize}")
        parallelism = (f"batch sharded over {world} GPUs (distributed.svdvals_sharded: one NCCL all-gather "
                       "of the values per step)" if world > 1 else "1 GPU")

        def step(inp, timers=None):
            if world > 1 and timers is None:
                return D.svdvals_sharded(cfg=cfg, backend=be, batch=total_units, make_shard=lambda a, b: inp)
            return call(inp, timers)

    for _ in range(max(args.warmup, 1)):
        step(x)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler()
    clocks.start()
    timers = {k: 0.0 for k in P.PHASE_KEYS}
    launches0 = L.bsvd_launch_counter()
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        step(x)
    e1.record(stream)
    torch.cuda.synchronize()
    launches = int(L.bsvd_launch_counter() - launches0)
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    # per-phase device timers from extra steps outside the timed region (the
    # timers add events and one synchronisation per phase)
    for _ in range(args.steps):
        step(x, timers)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    flops_step = flop_model(n) * total_units
    value = flops_step / (ms * 1e-3) / 1e12

    # ---- end to end through the public API with host buffers -------------
    e2e = None
    if not args.no_e2e:
        xh = x.cpu().pin_memory()
        step(xh)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ke = max(1, min(args.steps, 3))
        f0.record(stream)
        for _ in range(ke):
            step(xh)
        f1.record(stream)
        torch.cuda.synchronize()
        ems = f0.elapsed_time(f1) / ke
        te = torch.tensor([ems], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        ems = float(te.item())
        out_elem = 8 if dtype == torch.float64 else 4
        e2e = {"value": flops_step / (ems * 1e-3) / 1e12, "unit": "TFLOP/s",
               "ms_per_step": ems,
               "h2d_bytes_per_step": int(xh.numel() * xh.element_size()),
               "d2h_bytes_per_step": int(units * n * out_elem)}

    # ---- rooflines (phase spans from device events; per-kernel DRAM traffic
    # from the committed ncu capture of the same workload, profiles/traffic.json)
    hbm_gbs, smax, peak_src = measured_peaks()
    fp32_peak = 148 * 128 * 2 * smax * 1e6 / 1e12
    fp64_peak = fp32_peak / 2
    per = {k: v / args.steps * 1e3 for k, v in timers.items()}   # ms per step
    # panel chain and tensor-core updates overlap on two streams: stage 1's
    # wall time is the step minus the (serial) stage-2/3 spans
    stage1_ms = max(ms - per["bidiagonal"] - per["diagonal"], 1e-6)
    bw = cfg.tilesize
    npad = -(-n // bw) * bw
    fpk = fp64_peak if dtype == torch.float64 else fp32_peak
    fpk_src = (f"derived {'FP64' if dtype == torch.float64 else 'FP32'} FMA peak 148 SMs x "
               f"{64 if dtype == torch.float64 else 128} lanes x 2 x {smax:.0f} MHz "
               "(MEASURED_PEAKS.json has no CUDA-core FMA entry)")
    traffic = {}
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    except Exception:
        pass
    tc_on = dtype == torch.float32 and bw == 128 and os.environ.get("BSVD_FLAT_TC", "1") != "0"
    ach1 = flop_model(n) * units / (stage1_ms * 1e-3) / 1e12
    s1_model_bytes = 4.0 * npad ** 3 / (3.0 * bw) * (8 if dtype == torch.float64 else
                                                      2 if dtype == torch.float16 else 4) * units
    s1_traffic = traffic.get(f"stage1_step_n{n}") if wl == "single" else None
    phases = {
        "stage1": {"bound": "fma", "ms": stage1_ms, "achieved": ach1, "peak": fpk, "unit": "TFLOP/s", "frac": ach1 / fpk,
                   "kernel": ("stage 1: k_fpanel2 (cluster Householder panel) + k_tgemm (tcgen05 3xTF32 W = V^T X "
                              "and X -= V W2, TMA-fed) + k_tbuild + k_fw2x1" if tc_on else
                              "stage 1: k_fpanel2 + k_fgemm1/k_fgemm2 (FMA) + k_fgram + k_fw2x1"),
                   "peak_source": fpk_src, "model": "8/3 n^3 flops (the reference's count) over the stage-1 span",
                   "algorithmic_bytes": s1_model_bytes,
                   "bytes_model": "4 n^3/(3 ts) x elem: the trailing matrix read + written once per sweep side",
                   "traffic": s1_traffic},
    }
    # stage 2 chases in the compute precision (fp32 band for FP32/FP16, fp64 for FP64)
    belem = 8 if dtype == torch.float64 else 4
    algo_bytes = 2.0 * bw * npad * npad * belem * units
    ach2 = algo_bytes / (per["bidiagonal"] * 1e-3) / 1e9
    if bw > 64:
        chase_k = "k_chase2"
        chase_d = "k_chase2 (stage 2, carried-block cluster chase, one launch)"
    elif units >= 512:
        chase_k, chase_d = "k_chase_cta", "k_chase_cta (stage 2, one CTA per matrix, carried blocks in registers)"
    else:
        chase_k, chase_d = "k_chase", "k_chase (stage 2, pipelined cluster chase)"
    phases["bidiagonal"] = {"bound": "hbm", "kernel": chase_d, "ms": per["bidiagonal"],
                            "achieved": ach2, "peak": hbm_gbs, "unit": "GB/s", "frac": ach2 / hbm_gbs,
                            "peak_source": peak_src, "algorithmic_bytes": algo_bytes,
                            "model": f"touch model 2*bw*n^2*{belem} B per matrix (SURVEY.md 8(d)); the band "
                                     "(3b+1 rows) stays L2-resident, so the kernel is bound by its sweep "
                                     "dependency chain, not by DRAM",
                            "traffic": traffic.get(chase_k) if wl == "single" else None}
    # stage 3: the number of Sturm passes per value is data dependent; no flop
    # model -- time only
    phases["diagonal"] = {"bound": "latency", "kernel": "k_slice + k_values_u (stage 3, fp64 continuant Sturm counts + Laguerre)",
                          "ms": per["diagonal"], "achieved": None, "peak": None, "frac": None,
                          "traffic": traffic.get("k_values_u") if wl == "single" else None}
    # the required roofline object: the largest single kernel of the step (the
    # chase is one launch, timed live by its device events)
    roof = dict(phases["bidiagonal"])
    roof["kernel"] = chase_d

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        if wl == "single":
            cpu = cpu_baseline_fit(n)
        else:
            th = os.cpu_count() or 1
            dt = cpu_batch_sample(n, 16, th)
            cpu = {"value": 16 * flop_model(n) / dt / 1e12, "unit": "TFLOP/s", "cores": th, "kind": "port",
                   "extrapolated": False, "cpu_model": cpu_model(), "seconds": dt,
                   "sample": f"reference C port svdvals of 16 independent {n}^2 FP32 matrices, {th} OpenMP threads"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": {"fp32": "f32", "fp64": "f64", "fp16": "f16-storage/f32-compute"}[args.dtype],
            "data": "synthetic (N(0,1) random, seeded per rank; no dataset)",
            "config": {"workload": workload, "n": n, "tilesize": cfg.tilesize, "units_per_gpu": units,
                       "parallelism": parallelism,
                       "l2": "inputs larger than L2 (the padded working copy is rewritten every step)"},
            "stages_ms": per, "stage1_wall_ms": stage1_ms,
            "stage1_tflops": ach1,
            "roofline": roof, "phase_roofline": phases, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", choices=["single", "batch"], default=None,
                    help="default: single on 1 GPU, the sharded batch (configs[4]) on N > 1")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--ts", type=int, default=0)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--dtype", choices=["fp32", "fp64", "fp16"], default="fp32")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
