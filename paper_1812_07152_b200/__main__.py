"""``python -m paper_1812_07152_b200 <eval|inspect|bench> ...`` (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
