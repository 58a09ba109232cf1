"""lfem ORACLE — test infrastructure only (see lfem_oracle.cpp header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package.  The product package
paper_2605_14035_b200 never imports it.
"""
from .oracle import *  # noqa: F401,F403
