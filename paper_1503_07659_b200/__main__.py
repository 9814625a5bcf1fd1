"""``python -m paper_1503_07659_b200 ...``: see cli.py."""
import sys

from .cli import main

sys.exit(main())
