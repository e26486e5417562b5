cp paper_2508_06339_b200/lib/libbsvd.so /tmp/lib_default.so
for rep in 1 2; do
for u in 16 4; do
  if [ $u = 16 ]; then cp /tmp/lib_default.so paper_2508_06339_b200/lib/libbsvd.so; else cp probe_bin/pu$u/libbsvd.so paper_2508_06339_b200/lib/libbsvd.so; fi
  TAG=ulps$u python scripts/s3_time.py 8192
done
done
