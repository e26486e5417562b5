cp paper_2508_06339_b200/lib/libbsvd.so /tmp/libbsvd_epk1.so
for e in 1 2 4; do
  if [ $e != 1 ]; then cp probe_bin/epk$e/libbsvd.so paper_2508_06339_b200/lib/libbsvd.so; else cp /tmp/libbsvd_epk1.so paper_2508_06339_b200/lib/libbsvd.so; fi
  echo "EPK=$e"; python scripts/flat_check.py 2>&1 | grep "n=2048\|n=4096\|n=8192\|8192 err"
done
