"""⊤ count per valuation of one config-3 solve (PG_TRACE records): how much of V1's
later rounds is spent on ⊤ vertices. Usage: python scripts/top_probe.py [n d lo hi seed]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import pg_inputs as gi  # noqa: E402
from paper_1705_02313_b200 import Game  # noqa: E402

a = [int(x) for x in sys.argv[1:]] or [10_000_000, 32, 2, 5, 1]
g = gi.random_game(*a)
G = Game.from_game(g, trace=True)
r = G.solve()
t = G.get_trace()
for row in t:
    print(int(row[0]), int(row[3]), int(row[4]))
print({k: r.stats[k] for k in ("inner_iters", "outer_passes", "top_vertices") if k in r.stats})
