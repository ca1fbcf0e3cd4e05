"""Solve one game twice (warm-up, then traced) with the library's debug tracing
(PGSI_TRACE=1/2/3 in the environment: per-valuation lines / k_inc_iter phase times /
closure levels, on stderr). Usage: python scripts/trace_solve.py [n d lo hi seed]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import pg_inputs as gi  # noqa: E402
from paper_1705_02313_b200 import Game  # noqa: E402

a = [int(x) for x in sys.argv[1:]] or [10_000_000, 32, 2, 5, 1]
g = gi.random_game(*a)
G = Game.from_game(g)
G.solve()
print("---- traced solve", file=sys.stderr, flush=True)
r = G.solve()
print({k: r.stats[k] for k in ("inner_iters", "outer_passes", "inc_valuations", "ms_call")})
