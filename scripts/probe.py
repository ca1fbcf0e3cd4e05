"""Quick perf probe: load + solve configs with phase timing (not a bench number)."""
import sys, time, json
import numpy as np
sys.path.insert(0, "/root/repo")
import pg_inputs as gi
from paper_1705_02313_b200 import Game
import torch

for (n, d) in [(1_000_000, 16), (10_000_000, 32)]:
    t = time.time(); g = gi.random_game(n, d, 2, 5, 1); tg = time.time() - t
    t = time.time(); G = Game.from_game(g, phase_timing=True); tl = time.time() - t
    for rep in range(2):
        t = time.time(); r = G.solve(); ts = time.time() - t
        s = r.stats
        print(json.dumps({"n": n, "d": d, "gen_s": round(tg, 2), "load_s": round(tl, 2), "solve_s": round(ts, 4),
              "vals_per_s": n * s["inner_iters"] / ts, **{k: (round(v, 3) if isinstance(v, float) else v) for k, v in s.items()}}))
    del G
