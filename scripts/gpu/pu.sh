cp paper_2508_06339_b200/lib/libbsvd.so /tmp/lib_default.so
for u in 16 4 2; do
  if [ $u = 16 ]; then cp /tmp/lib_default.so paper_2508_06339_b200/lib/libbsvd.so; else cp probe_bin/pu$u/libbsvd.so paper_2508_06339_b200/lib/libbsvd.so; fi
  BSVD_S3_STATS=gpurun_out/s3_pu$u.bin python scripts/prof_one.py 8192
  echo "ulps=$u"; python scripts/values_check.py 2>&1 | tail -2
done
