mkdir -p gpurun_out
S3_WORST=1 python scripts/s3_stats.py 8192 u 4
python scripts/s3_time.py 8192 4 u
python scripts/s3_time.py 16384 4 u
