"""V2 design comparison: every valuation from scratch (PG_NO_INCREMENTAL)
with per-phase CUDA events, design S (depth-strided splitters + walks, the default) vs
design W (Wyllie over full d-vector rows, PGSI_V2_DESIGN=W), on config 3 and F_deep(4M).
Prints ms per full V2 and the V2 share of the solve. Usage: python scripts/v2_designs.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import pg_inputs as gi  # noqa: E402
from paper_1705_02313_b200 import Game  # noqa: E402

games = [("cfg3", gi.random_game(10_000_000, 32, 2, 5, 1)), ("F_deep(4M)", gi.f_deep(4_000_000))]
for name, g in games:
    for design in ("S", "W"):
        os.environ["PGSI_V2_DESIGN"] = design
        G = Game.from_game(g, incremental=False, phase_timing=True)
        G.solve()
        r = G.solve()
        st = r.stats
        print(f"{name} design {design}: V2 {st['ms_v2'] / max(st['n_v2'], 1):.3f} ms per valuation "
              f"({st['n_v2']} valuations), V1 {st['ms_v1'] / max(st['n_v1'], 1):.3f} ms, solve {st['ms_call']:.1f} ms "
              f"(wall), max depth {st['max_depth']}", flush=True)
        G.free()
