"""Solve time of the whole-solve cluster kernel against the multi-kernel path (device
loop) for mid-size games: where should pg_solve switch? Usage: python scripts/cluster_probe.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import pg_inputs as gi  # noqa: E402
from paper_1705_02313_b200 import Game  # noqa: E402

games = [("stair20k", gi.f_stair(20000))]
for n in (6_000, 12_000, 25_000, 50_000, 100_000):
    for d in (4, 8, 16):
        games.append((f"rand n={n} d={d}", gi.random_game(n, d, 2, 5, 1)))
games += [("ladder 40k", gi.ladder(40_000, 1)), ("elevator 10/8", gi.elevator(10, 8, 1))]
for name, g in games:
    row = [name]
    for cmax in ("0", ""):
        os.environ["PGSI_SMALL_MAX"] = "0"
        os.environ["PGSI_CLUSTER"] = "0" if cmax else "2"
        G = Game.from_game(g)
        for _ in range(2):
            G.solve()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(3):
            r = G.solve()
        e1.record()
        torch.cuda.synchronize()
        row.append(f"{'multi' if cmax else 'cluster' if r.stats['cluster_solves'] else 'multi(nofit)'} "
                   f"{e0.elapsed_time(e1) / 3:.3f} ms")
        G.free()
    print(" | ".join(row), f"n'={G.n_internal} inner={r.stats['inner_iters']}", flush=True)
