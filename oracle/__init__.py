"""fp64 CPU oracle for the SANTA / S^2ANTA decode hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  The product package never does.
"""
from .santa_oracle import *  # noqa: F401,F403
from . import santa_oracle  # noqa: F401
