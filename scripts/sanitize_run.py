"""One solve (plus a valuation and a best response) through the C ABI, checked
against the oracle, for compute-sanitizer runs (scripts/sanitize.sh).
Usage: python scripts/sanitize_run.py N D [multikernel|cluster [devloop]]
(devloop: the solve runs as the device-resident CUDA graph, PGSI_DEVICE_LOOP=2)"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
n, d = int(sys.argv[1]), int(sys.argv[2])
if len(sys.argv) > 3 and sys.argv[3] in ("multikernel", "cluster"):
    os.environ["PGSI_SMALL_MAX"] = "0"
    os.environ["PGSI_HOST_LOAD_MAX"] = "0"
    os.environ["PGSI_CLUSTER"] = "0" if sys.argv[3] == "multikernel" else "2"
if len(sys.argv) > 4 and sys.argv[4] == "devloop":
    os.environ["PGSI_DEVICE_LOOP"] = "2"
import pg_inputs as gi  # noqa: E402
from oracle import Oracle  # noqa: E402
from paper_1705_02313_b200 import Game  # noqa: E402

g = gi.random_game(n, d, 2, 5, 1)
o = Oracle(g)
ref = o.solve()
G = Game.from_game(g)
r = G.solve(want_val=True)
assert r.stats["inner_iters"] == ref.inner_iters and r.stats["outer_passes"] == ref.outer_passes
for k in ("winner", "sigma", "tau"):
    assert np.array_equal(getattr(r, k), getattr(ref, k)), k
assert np.array_equal(r.val, ref.val)
s = ref.succ_int
val, top, cd = G.valuate(s)
assert np.array_equal(top, ref.top_int)
tau, _, _, inner = G.best_response(s)
print(f"ok n={n} d={d} inner={r.stats['inner_iters']} outer={r.stats['outer_passes']} "
      f"inc={r.stats['inc_valuations']} small={r.stats['small_solves']}")
