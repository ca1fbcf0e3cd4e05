"""Compact-prefix width probe: solve config 3 with 1-7 stored (column, count) pairs and
report the undecided compares (full re-walk compares) and the solve time."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import pg_inputs as gi  # noqa: E402
from paper_1705_02313_b200 import Game  # noqa: E402
g = gi.random_game(10_000_000, 32, 2, 5, 1)
for pp in (7, 5, 3, 2):
    G = Game.from_game(g, prefix_pairs=pp)
    G.solve()
    r = G.solve()
    print(pp, {k: r.stats.get(k) for k in ("inner_iters", "full_compares", "prefix_gathers", "ms_call")}, flush=True)
    G.free()
