mkdir -p gpurun_out
python scripts/s3_stats.py 8192 1 4
python scripts/s3_time.py 8192 1 4
python scripts/s3_time.py 16384 1 4
python scripts/s3_time.py 1024 1 4
python -m pytest tests -m gpu -x -q 2>&1 | tail -4
