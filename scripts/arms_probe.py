"""Table 2 analogue probe (not a bench number): SI vs SI-Reset vs Bellman-Ford best
responses on a synthetic game; per arm solve time, iterations, BF round GB/s."""
import json
import sys
import time

sys.path.insert(0, "/root/repo")
import pg_inputs as gi  # noqa: E402
from paper_1705_02313_b200 import Game  # noqa: E402

n, d = int(sys.argv[1]), int(sys.argv[2])
arms = sys.argv[3].split(",") if len(sys.argv) > 3 else ["si", "si_reset", "bf"]
g = gi.random_game(n, d, 2, 5, 1)
for arm in arms:
    G = Game.from_game(g, phase_timing=True, best_response=arm)
    t = time.perf_counter()
    r = G.solve()
    s = r.stats
    out = {"arm": arm, "n": n, "d": d, "wall_s": round(time.perf_counter() - t, 3),
           "ms_call": round(s["ms_call"], 2), "inner": s["inner_iters"], "outer": s["outer_passes"]}
    if arm == "bf":
        out.update(bf_ms_per_round=round(s["ms_bf"] / max(s["n_bf"], 1), 4),
                   bf_GBps=round(s["bytes_bf"] / (s["ms_bf"] / 1e3) / 1e9, 1) if s["ms_bf"] else None,
                   bf_MB_per_round=round(s["bytes_bf"] / max(s["n_bf"], 1) / 1e6, 1))
    print(json.dumps(out), flush=True)
    G.free()
