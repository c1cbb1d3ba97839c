"""`levlu` alias of the B200 package (test harness only).

Binds the reference's import name to paper_1908_00204_b200 so the
reference's own test suite (/root/reference/pkg/tests, copied to the
git-ignored baseline/_ref/tests for the GPU box) runs unmodified against
the drop-in: PYTHONPATH=tools/levlu_alias:. python -m pytest baseline/_ref/tests
"""

from paper_1908_00204_b200 import *  # noqa: F401,F403
from paper_1908_00204_b200 import __version__  # noqa: F401
from paper_1908_00204_b200 import cli, depgraph, numeric, resource, sparse, symbolic  # noqa: F401
