"""`levlu.cli` alias (see levlu/__init__.py here)."""

from paper_1908_00204_b200.cli import *  # noqa: F401,F403
from paper_1908_00204_b200.cli import main  # noqa: F401
