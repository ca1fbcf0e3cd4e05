"""B200-native greedy all-switches strategy improvement for parity games
(Fearnley, arXiv 1705.02313): valuation + all-switches hot path in CUDA for
sm_100a behind the C ABI of ``include/pg.h``; this package is its thin binding."""
from .pg import (  # noqa: F401
    Game, PGError, Stats, Options, SolveResult, load_library, version, LIB_PATH,
    PG_SINK, PG_NONE, parse_pgsolver, format_solution, verify_solution, ParsedGame, dist_unique_id,
)
