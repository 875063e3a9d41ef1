"""CPU oracle for the QVA hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  The product path (paper_2110_03963_b200) never does,
and the two share no code.

Parity status of each function is listed in DESIGN.md "Oracle pins"; every function
here is pinned by a `-m "not gpu"` test in tests/test_oracle_pins.py.
"""
from .oracle import *  # noqa: F401,F403
