"""End-to-end breakdown of config 3 through the public API with pinned host buffers:
pg_load (H2D + device transform), the first and second pg_solve (with the outputs copied
back) and pg_free, four times. Usage: python scripts/e2e_probe.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import pg_inputs as gi
from paper_1705_02313_b200 import Game
g = gi.random_game(10_000_000, 32, 2, 5, 1)
def pinned(a):
    t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory(); return t, t.numpy()
keep = [pinned(g.row_ptr), pinned(g.col), pinned(g.owner), pinned(g.priority)]
rp, col, own, pri = [k[1] for k in keep]
n = g.n
hw = torch.empty(n, dtype=torch.uint8).pin_memory().numpy()
hs = torch.empty(n, dtype=torch.int32).pin_memory().numpy()
ht = torch.empty(n, dtype=torch.int32).pin_memory().numpy()
s = torch.cuda.Stream()
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    G = Game(n, rp, col, own, pri, device=0, stream=s.cuda_stream)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    r = G.solve(out=(hw, hs, ht, None))
    torch.cuda.synchronize(); t2 = time.perf_counter()
    r2 = G.solve(out=(hw, hs, ht, None))
    torch.cuda.synchronize(); t3 = time.perf_counter()
    G.free()
    torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"load {1e3*(t1-t0):.2f} ms  solve1 {1e3*(t2-t1):.2f} (call {r.stats.get('ms_call')})  solve2 {1e3*(t3-t2):.2f}  free {1e3*(t4-t3):.2f}", flush=True)
