"""Tune incremental thresholds (not a bench number): solve time per setting."""
import os, sys, json, subprocess
sys.path.insert(0, "/root/repo")
settings = [("48", "8", "64"), ("24", "8", "64"), ("32", "16", "64"), ("64", "8", "64"), ("48", "8", "32"), ("48", "8", "128"), ("48", "4", "32")]
code = r'''
import sys, torch
sys.path.insert(0, "/root/repo")
import pg_inputs as gi
from paper_1705_02313_b200 import Game
g = gi.random_game(int(sys.argv[1]), int(sys.argv[2]), 2, 5, 1)
s = torch.cuda.current_stream()
G = Game.from_game(g, stream=s.cuda_stream, device_ptrs=True)
n = g.n
out = (torch.empty(n, dtype=torch.uint8, device="cuda"), torch.empty(n, dtype=torch.int32, device="cuda"), torch.empty(n, dtype=torch.int32, device="cuda"), None)
for _ in range(2): G.solve(out=out)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record(s)
for _ in range(3): r = G.solve(out=out)
e1.record(s); torch.cuda.synchronize()
print(e0.elapsed_time(e1) / 3, r.stats["inc_valuations"], r.stats["inc_aborts"])
'''
for lv, dd, sd in settings:
    env = dict(os.environ, PGSI_INC_MAX_LEVELS=lv, PGSI_INC_DIRTY_DIV=dd, PGSI_INC_S_DIV=sd)
    out = subprocess.run([sys.executable, "-c", code, sys.argv[1], sys.argv[2]], env=env, capture_output=True, text=True)
    print(json.dumps({"levels": lv, "dirty_div": dd, "s_div": sd, "result": out.stdout.strip() or out.stderr[-300:]}), flush=True)
