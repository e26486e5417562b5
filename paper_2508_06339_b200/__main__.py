"""python -m paper_2508_06339_b200 {svdvals,accuracy,bench,tune} ... (cli.py)."""
import sys

from .cli import main

sys.exit(main())
