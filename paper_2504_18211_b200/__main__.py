"""python -m paper_2504_18211_b200 {trial,sweep,selftest} ... (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
