"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package. It shares no code with the
CUDA path (paper_2604_08075_b200/, include/). See fleet_oracle.c's header.
"""
from .oracle import *  # noqa: F401,F403
