"""Wall time of the first and later pg_solve calls on a handle (the first one builds
and instantiates the device-loop graph). Usage: python scripts/graph_build_probe.py [n]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import pg_inputs as gi  # noqa: E402
from paper_1705_02313_b200 import Game  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
g = gi.random_game(n, 32, 2, 5, 1)
for loop in ("1", "0"):
    os.environ["PGSI_DEVICE_LOOP"] = loop
    for rep in range(2):
        t0 = time.perf_counter()
        G = Game.from_game(g)
        t1 = time.perf_counter()
        times = []
        for _ in range(3):
            a = time.perf_counter()
            r = G.solve()
            times.append(1000 * (time.perf_counter() - a))
        print(f"loop={loop} load {1000*(t1-t0):.1f} ms, solves {['%.2f' % x for x in times]} ms, "
              f"device_loop={r.stats['device_loop_solves']}")
        G.free()
