timeout 900 python scripts/traffic_capture.py 8192 > gpurun_out/traffic.log 2>&1; tail -12 gpurun_out/traffic.log
timeout 600 python bench.py > gpurun_out/bench_single.json 2> gpurun_out/bench_single.err; tail -c 600 gpurun_out/bench_single.err
timeout 600 python bench.py --workload batch --no-cpu > gpurun_out/bench_batch.json 2> gpurun_out/bench_batch.err; tail -c 400 gpurun_out/bench_batch.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 400 gpurun_out/bench_ref.err
