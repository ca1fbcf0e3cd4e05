"""CPU oracle (TEST INFRASTRUCTURE ONLY).

A plain, slow, single-threaded C implementation of Fearnley's greedy
all-switches strategy improvement (arXiv 1705.02313, Algorithm 1)
with the obvious sequential valuation. See ``pg_oracle.c``'s
header for the paper passages each function follows.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package. The CUDA product path
(``paper_1705_02313_b200``) never imports it and shares no code with it.
"""
from .oracle import Oracle, OracleError, build_oracle, oracle_lib_path  # noqa: F401
