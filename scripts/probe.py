"""Perf probe (not a bench number): per-valuation walk statistics."""
import sys, time, json
sys.path.insert(0, "/root/repo")
import numpy as np
import pg_inputs as gi
from paper_1705_02313_b200 import Game
n, d = int(sys.argv[1]), int(sys.argv[2])
g = gi.random_game(n, d, 2, 5, 1)
G = Game.from_game(g, phase_timing=True)
owner = None
r = G.solve()
s = r.stats
print(json.dumps({k: s[k] for k in ("inner_iters", "walk_steps", "top_vertices", "v1_rounds", "max_depth", "ms_v1", "ms_v2", "ms_odd", "ms_even", "ms_call")}))
print("mean walk steps per vertex per valuation", s["walk_steps"] / s["inner_iters"] / G.n_internal)
print("mean top fraction", s["top_vertices"] / s["inner_iters"] / G.n_internal)
