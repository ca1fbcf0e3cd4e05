"""Seeded synthetic parity-game generators.

This package is shared by the CPU oracle tests and the CUDA path's tests/bench:
it only *produces inputs* (CSR edges, owner, priority). It contains none of the
method's arithmetic (no valuation, comparison, switching or preprocessing), so
sharing it does not couple the oracle to the CUDA path.

All games are returned as a :class:`Game` in the boundary's layout
(``include/pg.h``, ``pg_load``): ``row_ptr`` int64[n+1], ``col`` int32[m],
``owner`` uint8[n] (0 = Even, 1 = Odd), ``priority`` int32[n] (>= 0).
"""
from .games import (  # noqa: F401
    Game,
    mix64,
    counter_hash,
    random_game,
    f_stair,
    f_stairs,
    f_deep,
    f_oddchain,
    ladder,
    hanoi,
    elevator,
    fixture_g2,
    from_adjacency,
    pgsolver_text,
    parse_pgsolver,
)
