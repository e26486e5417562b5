# A/B: continuant (default build) vs ratio-form Sturm counts, then the GPU suite
mkdir -p gpurun_out
cp paper_2508_06339_b200/lib/libbsvd.so /tmp/lib_default.so
for rep in 1 2; do
  cp probe_bin/ratio/libbsvd.so paper_2508_06339_b200/lib/libbsvd.so; TAG=ratio python scripts/s3_time.py 8192
  cp /tmp/lib_default.so paper_2508_06339_b200/lib/libbsvd.so; TAG=cont python scripts/s3_time.py 8192
done
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
