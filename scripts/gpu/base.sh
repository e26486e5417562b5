set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/base_bench.json 2>gpurun_out/base_bench.err
tail -c 600 gpurun_out/base_bench.json
