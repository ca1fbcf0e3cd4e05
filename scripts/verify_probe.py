"""Timing probe (not a bench number): host vs GPU solution verifier on a solved game."""
import sys
import time

sys.path.insert(0, "/root/repo")
import pg_inputs as gi  # noqa: E402
from paper_1705_02313_b200 import Game, verify_solution  # noqa: E402

n, d = int(sys.argv[1]), int(sys.argv[2])
g = gi.random_game(n, d, 2, 5, 1)
r = Game.from_game(g).solve()
for dev in (None, 0, 0):
    t = time.perf_counter()
    ok, w, msg = verify_solution(g, r.winner, r.sigma, r.tau, device=dev)
    print(f"n={n} d={d} {'host' if dev is None else 'gpu '} ok={ok} {time.perf_counter() - t:.2f} s {msg[:60]}", flush=True)
