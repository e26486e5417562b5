timeout 600 python scripts/flat_check.py 2>&1 | tail -20
BSVD_FPANEL_V1=1 timeout 300 python scripts/flat_check.py 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
