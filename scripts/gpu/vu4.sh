mkdir -p gpurun_out
cp paper_2508_06339_b200/lib/libbsvd.so /tmp/lib_default.so
for v in default sided1 t18 t30; do
  if [ $v = default ]; then cp /tmp/lib_default.so paper_2508_06339_b200/lib/libbsvd.so; else cp probe_bin/$v/libbsvd.so paper_2508_06339_b200/lib/libbsvd.so; fi
  echo "== $v"
  python scripts/s3_stats.py 8192 u
  python scripts/s3_time.py 8192 u
  python scripts/s3_time.py 16384 u
done
cp /tmp/lib_default.so paper_2508_06339_b200/lib/libbsvd.so
