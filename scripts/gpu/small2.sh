# small-n stage 1: split counts + panel rows per thread
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python scripts/small_n.py 2>&1 | tail -6
for r in 4 8; do echo "RPT=$r"; BSVD_FLAT_RPT=$r python scripts/small_n.py 2>&1 | head -3; done
