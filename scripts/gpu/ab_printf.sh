cp paper_2508_06339_b200/lib/libbsvd.so /tmp/lib_default.so
for rep in 1 2; do
cp /tmp/lib_default.so paper_2508_06339_b200/lib/libbsvd.so; TAG=printf python scripts/s3_time.py 8192 u
cp probe_bin/noprintf/libbsvd.so paper_2508_06339_b200/lib/libbsvd.so; TAG=noprintf python scripts/s3_time.py 8192 u
done
cp /tmp/lib_default.so paper_2508_06339_b200/lib/libbsvd.so
