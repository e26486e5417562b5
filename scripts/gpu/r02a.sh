set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python scripts/flat_check.py > gpurun_out/flat_check.log 2>&1; tail -30 gpurun_out/flat_check.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -15 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench.json 2>gpurun_out/bench.err
tail -c 3000 gpurun_out/bench.json
