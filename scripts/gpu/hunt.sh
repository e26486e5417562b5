mkdir -p gpurun_out
python scripts/s3_worst_bench.py 16384 2>/dev/null | head -4
python scripts/s3_worst_bench.py 8192 2>/dev/null | head -3
python scripts/s3_stats.py 8192 u
python scripts/s3_stats.py 16384 u
python scripts/s3_time.py 8192 u 1
python scripts/s3_time.py 16384 u
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
