"""CPU oracle for the multinomial-logit Newton-Raphson hot path (TEST INFRASTRUCTURE).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import this package.  The product path
(`paper_1404_3177_b200`) never imports it and shares no code with it.
"""
from .mnl_oracle import *  # noqa: F401,F403
