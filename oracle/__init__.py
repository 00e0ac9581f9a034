"""CPU oracles for the multinomial-logit Newton-Raphson hot path (TEST INFRASTRUCTURE).

Two independent codings of the same plain definition:
  oracle.mnl_oracle  -- numpy (re-exported here)
  oracle.coracle     -- ctypes adapter of liboracle.so (oracle/oracle.c, plain C + OpenMP,
                        O(n_p^2) memory; exports oracle_mnl_eval / oracle_mnl_newton_fit)

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import this package.  The product path
(`paper_1404_3177_b200`) never imports it and shares no code with it.
"""
from .mnl_oracle import *  # noqa: F401,F403
