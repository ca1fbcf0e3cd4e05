"""Solve time vs splitter stride K (not a bench number)."""
import sys, torch
sys.path.insert(0, "/root/repo")
import pg_inputs as gi
from paper_1705_02313_b200 import Game
g = gi.random_game(int(sys.argv[1]), int(sys.argv[2]), 2, 5, 1)
s = torch.cuda.current_stream()
n = g.n
out = (torch.empty(n, dtype=torch.uint8, device="cuda"), torch.empty(n, dtype=torch.int32, device="cuda"),
       torch.empty(n, dtype=torch.int32, device="cuda"), None)
for k in [int(x) for x in sys.argv[3].split(",")]:
    G = Game.from_game(g, stream=s.cuda_stream, device_ptrs=True, splitter_k=k, phase_timing=True)
    for _ in range(2): G.solve(out=out)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(s)
    for _ in range(3): r = G.solve(out=out)
    e1.record(s); torch.cuda.synchronize()
    st = r.stats
    print(f"K={k}: {e0.elapsed_time(e1)/3:.2f} ms  v2/launch {st['ms_v2']/max(st['n_v2'],1):.3f}  v1/launch {st['ms_v1']/max(st['n_v1'],1):.3f}", flush=True)
    G.free()
