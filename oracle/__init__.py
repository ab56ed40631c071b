"""ORACLE — test infrastructure only (see ppca_oracle.py header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  The product path never does.
"""
from .ppca_oracle import *  # noqa: F401,F403
from . import ppca_oracle  # noqa: F401
