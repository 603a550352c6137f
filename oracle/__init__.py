"""CPU oracle for the coophash hot path -- TEST INFRASTRUCTURE ONLY.

Never imported by the product package ``paper_2009_07914_b200``.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU leg use it, as
the checker / CPU baseline.  See ``oracle.c`` for the reference citations and
``tests/test_oracle.py`` for how it is pinned to the reference's own outputs.
"""
from .oracle import *  # noqa: F401,F403
