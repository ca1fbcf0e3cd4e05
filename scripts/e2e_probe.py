"""e2e breakdown probe (not a bench number): pinned H2D of the raw CSR alone,
pg_load (its own H2D + GPU transform), pg_solve, D2H of winner/σ/τ."""
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import pg_inputs as gi  # noqa: E402
from paper_1705_02313_b200 import Game  # noqa: E402

g = gi.random_game(10_000_000, 32, 2, 5, 1)
pin = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (g.row_ptr, g.col, g.owner, g.priority)]
dev = [torch.empty_like(p, device="cuda") for p in pin]
for _ in range(2):
    for p, d in zip(pin, dev):
        d.copy_(p, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for p, d in zip(pin, dev):
    d.copy_(p, non_blocking=True)
torch.cuda.synchronize()
h2d = (time.perf_counter() - t) * 1e3
nb = sum(p.numel() * p.element_size() for p in pin)
print(f"H2D {nb / 1e6:.0f} MB pinned: {h2d:.2f} ms ({nb / h2d / 1e6:.1f} GB/s)")
rp, col, own, pri = [p.numpy() for p in pin]
hw = torch.empty(g.n, dtype=torch.uint8).pin_memory().numpy()
hs = torch.empty(g.n, dtype=torch.int32).pin_memory().numpy()
ht = torch.empty(g.n, dtype=torch.int32).pin_memory().numpy()
for it in range(4):
    t0 = time.perf_counter()
    G = Game(g.n, rp, col, own, pri)
    t1 = time.perf_counter()
    r = G.solve(out=(hw, hs, ht, None))
    t2 = time.perf_counter()
    G.free()
    t3 = time.perf_counter()
    print(f"iter {it}: pg_load {1e3 * (t1 - t0):.2f} ms (ms_load {r.stats['ms_load']:.2f}), solve+D2H {1e3 * (t2 - t1):.2f} ms, free {1e3 * (t3 - t2):.2f} ms")
