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

`--impl reference` times the reference's CPU path -- the bit-exact C port of
the reference (oracle/, "kind": "port"; the reference is Python+numba with no
compiled core to link) -- on the host's cores, rank 0 only, on a bounded
sample of the same workload (one 2048 x 2048 FP32 matrix, ts = 128 per step).
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


def cpu_baseline_sample(threads=None):
    """Time the reference's CPU path (C port, all host threads) on the bounded
    sample; returns (TFLOP/s, seconds, threads, description)."""
    import numpy as np
    from oracle import oracle as O
    O.lib()
    th = threads or os.cpu_count() or 1
    O.set_num_threads(th)
    a = np.random.default_rng(0xBE7C).standard_normal((CPU_SAMPLE_N, CPU_SAMPLE_N)).astype(np.float32)
    t0 = time.perf_counter()
    O.svdvals(a, 128)
    dt = time.perf_counter() - t0
    desc = (f"reference C port (oracle/bsvd_oracle.c, bit-exact to bandsvd) svdvals of one "
            f"{CPU_SAMPLE_N}x{CPU_SAMPLE_N} FP32 N(0,1) matrix, ts=128, {th} OpenMP threads; "
            f"TFLOP/s on the 8/3 n^3 model of the sample")
    return flop_model(CPU_SAMPLE_N) / dt / 1e12, dt, th, desc


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    for _ in range(args.warmup):
        cpu_baseline_sample()
    vals, secs = [], []
    th = os.cpu_count() or 1
    for _ in range(args.steps):
        v, dt, th, desc = cpu_baseline_sample()
        vals.append(v)
        secs.append(dt)
    v = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.median(secs) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (N(0,1), seeded)",
        "config": {"workload": f"bounded CPU sample of configs[1]: {CPU_SAMPLE_N}x{CPU_SAMPLE_N} FP32 "
                               "(the GPU arm runs 8192x8192 FP32, ts=128)",
                   "n": CPU_SAMPLE_N, "tilesize": 128},
        "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": th, "kind": "port", "sample": desc},
        "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


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

    if args.workload == "single":
        n = args.n or 8192
        cfg = P.KernelConfig.for_size(n) if not args.ts else P.KernelConfig(tilesize=args.ts)
        x = torch.randn((n, n), generator=gen, device=dev, dtype=torch.float32).to(dtype)
        units = 1
        call = lambda inp, timers=None: P.svdvals(inp, cfg, be, timers)
        workload = (f"configs[1]: one {n}x{n} {args.dtype.upper()} N(0,1) matrix per GPU, svdvals "
                    f"(all singular values), default tiles ts={cfg.tilesize}")
    else:
        n = args.n or 512
        total = args.batch or 4096
        per = total // world
        cfg = P.KernelConfig.for_size(n) if not args.ts else P.KernelConfig(tilesize=args.ts)
        x = torch.randn((per, n, n), generator=gen, device=dev, dtype=torch.float32).to(dtype)
        units = per
        call = lambda inp, timers=None: P.svdvals_batched(inp, cfg, be, timers)
        workload = (f"configs[4]: batch of {total} independent {n}x{n} {args.dtype.upper()} matrices "
                    f"sharded {per} per GPU, ts={cfg.tilesize}")

    def step(inp, timers=None):
        vals = call(inp, timers)
        if world > 1:
            vt = vals if isinstance(vals, torch.Tensor) else torch.from_numpy(vals).to(dev)
            out = [torch.empty_like(vt) for _ in range(world)]
            dist.all_gather(out, vt.contiguous())
            return out
        return vals

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
    flops_step = flop_model(n) * units * world
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

    # ---- roofline of the dominant phase (device events over the timed steps)
    hbm_gbs, smax, peak_src = measured_peaks()
    fp32_peak = 148 * 128 * 2 * smax * 1e6 / 1e12
    fp64_peak = fp32_peak / 2
    per = {k: v / args.steps * 1e3 for k, v in timers.items()}   # ms per step
    # panel and trailing overlap on two streams: stage 1's wall time is the step
    # minus the (serial) stage-2/3 spans
    stage1_ms = max(ms - per["bidiagonal"] - per["diagonal"], 1e-6)
    walls = {"stage1": stage1_ms, "bidiagonal": per["bidiagonal"], "diagonal": per["diagonal"]}
    dom = max(walls, key=walls.get)
    bw = cfg.tilesize
    npad = -(-n // bw) * bw
    fpk = fp64_peak if dtype == torch.float64 else fp32_peak
    fpk_src = (f"derived {'FP64' if dtype == torch.float64 else 'FP32'} FMA peak 148 SMs x "
               f"{64 if dtype == torch.float64 else 128} lanes x 2 x {smax:.0f} MHz "
               "(MEASURED_PEAKS.json has no CUDA-core FMA entry)")
    ach1 = flop_model(n) * units / (stage1_ms * 1e-3) / 1e12
    phases = {
        "stage1": {"bound": "fma", "kernel": "stage 1 (k_panel_leaf2/k_panel_tt + k_leaf2_u/k_node_tu + k_apply_leaf2/k_apply_tt on 3 streams)",
                   "achieved": ach1, "peak": fpk, "unit": "TFLOP/s", "frac": ach1 / fpk,
                   "peak_source": fpk_src, "model": "8/3 n^3 flops (the reference's count)", "traffic": None},
    }
    # stage 2 chases in the compute precision (fp32 band for FP32/FP16, fp64 for FP64)
    belem = 8 if dtype == torch.float64 else 4
    algo_bytes = 2.0 * bw * npad * npad * belem * units
    ach2 = algo_bytes / (per["bidiagonal"] * 1e-3) / 1e9
    if bw > 64:
        chase_k = "k_chase2 (stage 2, carried-block cluster chase, one launch)"
    elif units >= 512:
        chase_k = "k_chase_cta (stage 2, one CTA per matrix, carried blocks in registers)"
    else:
        chase_k = "k_chase (stage 2, pipelined cluster chase)"
    phases["bidiagonal"] = {"bound": "hbm", "kernel": chase_k,
                            "achieved": ach2, "peak": hbm_gbs, "unit": "GB/s", "frac": ach2 / hbm_gbs,
                            "peak_source": peak_src, "algorithmic_bytes": algo_bytes,
                            "model": f"touch model 2*bw*n^2*{belem} B per matrix (SURVEY.md 8(d))", "traffic": None}
    # stage 3: counted Sturm steps are not fixed; report time against the FP64 pipe
    # on a 64-count-per-value model of plain bisection (the work it replaces)
    algo3 = units * n * 64 * 2 * npad * 10.0
    ach3 = algo3 / (per["diagonal"] * 1e-3) / 1e12
    phases["diagonal"] = {"bound": "fma", "kernel": "k_slice + k_values (stage 3)", "achieved": ach3,
                          "peak": fp64_peak, "unit": "TFLOP/s", "frac": ach3 / fp64_peak,
                          "peak_source": "derived FP64 FMA peak",
                          "model": "64 Sturm counts x 2n steps x 10 flops per value (bisection-equivalent)",
                          "traffic": None}
    roof = dict(phases[dom])
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof):
        try:
            tr = json.load(open(prof))
            roof["traffic"] = tr.get(roof["kernel"].split()[0])
            for ph in phases.values():
                ph["traffic"] = tr.get(ph["kernel"].split()[0])
        except Exception:
            pass

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, dt, th, desc = cpu_baseline_sample()
        cpu = {"value": v, "unit": "TFLOP/s", "cores": th, "kind": "port", "sample": desc,
               "seconds": dt}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": {"fp32": "f32", "fp64": "f64", "fp16": "f16-storage/f32-compute"}[args.dtype],
            "data": "synthetic (N(0,1) random, seeded per rank; no dataset)",
            "config": {"workload": workload, "n": n, "tilesize": cfg.tilesize, "units_per_gpu": units,
                       "parallelism": f"replicas x{world} (values all-gathered over NCCL)" if world > 1 else "1 GPU",
                       "l2": "inputs larger than L2 (the padded working copy is rewritten every step)"},
            "stages_ms": per, "stage1_wall_ms": stage1_ms,
            "stage1_tflops": flop_model(n) * units / (stage1_ms * 1e-3) / 1e12,
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
    ap.add_argument("--workload", choices=["single", "batch"], default="single")
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
