"""Crossover probe (not a bench number): whole-solve single-block kernel vs the
multi-kernel loop on random games of growing size. Usage: small_probe.py d"""
import os
import sys
import time

sys.path.insert(0, "/root/repo")
import pg_inputs as gi  # noqa: E402
from paper_1705_02313_b200 import Game  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 16
for n in (1000, 3000, 6000, 12000, 25000, 50000, 100000):
    g = gi.random_game(n, d, 2, 5, 1)
    out = []
    for sm in ("0", str(1 << 30)):
        os.environ["PGSI_SMALL_MAX"] = sm
        G = Game.from_game(g)
        for _ in range(2):
            G.solve()
        t = time.perf_counter()
        for _ in range(5):
            r = G.solve()
        out.append((time.perf_counter() - t) / 5 * 1e3)
        G.free()
    print(f"n={n} n'={G.n_internal} d={d} inner={r.stats['inner_iters']} multi={out[0]:.3f} ms small={out[1]:.3f} ms", flush=True)
