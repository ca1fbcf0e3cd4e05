"""Perf probe (not a bench number): phase times and walk statistics per config."""
import sys, time, json
sys.path.insert(0, "/root/repo")
import pg_inputs as gi
from paper_1705_02313_b200 import Game
n, d = int(sys.argv[1]), int(sys.argv[2])
ks = [int(k) for k in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0]
g = gi.random_game(n, d, 2, 5, 1)
for k in ks:
    G = Game.from_game(g, phase_timing=True, splitter_k=k)
    G.solve()
    r = G.solve()
    s = r.stats
    it = s["inner_iters"]
    print(json.dumps({"K": k, "ms_call": round(s["ms_call"], 2), "inner": it,
                      "v1_ms": round(s["ms_v1"] / it, 4), "v2_ms": round(s["ms_v2"] / it, 4),
                      "odd_ms": round(s["ms_odd"] / it, 4), "even_ms": round(s["ms_even"] / max(s["n_even"], 1), 4),
                      "split_vals": s["v2_split_valuations"], "steps_per_v": round(s["walk_steps"] / it / G.n_internal, 3),
                      "full_cmp": s["full_compares"]}))
    G.free()
