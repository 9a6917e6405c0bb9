"""``python -m paper_2209_06916_b200 solve|iters ...`` (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
