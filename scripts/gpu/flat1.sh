timeout 600 python scripts/flat_check.py 2>&1 | tail -40
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
