timeout 1200 python scripts/verify_configs.py > gpurun_out/verify.log 2>&1; tail -8 gpurun_out/verify.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench_single.json 2> gpurun_out/bench_single.err; tail -c 300 gpurun_out/bench_single.json
python - <<'PY'
import sys, time, torch
sys.path.insert(0, '.')
import paper_2508_06339_b200 as P
for n, dt in ((16384, torch.float32), (4096, torch.float32), (8192, torch.float16)):
    a = torch.randn(n, n, device='cuda').to(dt)
    P.svdvals(a); torch.cuda.synchronize()
    tm = {k: 0.0 for k in P.PHASE_KEYS}
    t0 = time.perf_counter(); P.svdvals(a, timers=tm); torch.cuda.synchronize(); dt_s = time.perf_counter() - t0
    print(f"n={n} {dt}: {dt_s*1e3:.1f} ms  {8/3*n**3/dt_s/1e12:.2f} TF/s  stage1 {tm['panel']*1e3:.1f} chase {tm['bidiagonal']*1e3:.1f} values {tm['diagonal']*1e3:.1f}", flush=True)
PY
