"""CPU oracle for the Tokencake offload/upload hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import this package.
It shares no code with paper_2510_18586_b200 (the CUDA path) and never imports it.  See oracle/pool.py.
"""
from .pool import (ALLOC, FREE, PENDING, RESERVED, E_BUSY, E_HANDLE, E_INVAL, E_NOBLOCKS, E_NOHOST, OK,  # noqa: F401
                   BytesStore, OracleError, OraclePool, ProvStore)
