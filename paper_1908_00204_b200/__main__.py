"""`python -m paper_1908_00204_b200 factor|solve ...` (see cli.py)."""

import sys

from .cli import main

sys.exit(main())
