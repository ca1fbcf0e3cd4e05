"""Debug: incremental valuation vs from-scratch on small games (PGSI_VERIFY_INC=1)."""
import os, sys
os.environ["PGSI_VERIFY_INC"] = "1"
sys.path.insert(0, "/root/repo")
import numpy as np
import pg_inputs as gi
from oracle import Oracle
from paper_1705_02313_b200 import Game, PGError
for seed in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    g = gi.random_game(1000, 4, 2, 3, seed)
    ora = Oracle(g).solve()
    G = Game.from_game(g, max_inner=5000)
    try:
        r = G.solve()
        ok = r.stats["inner_iters"] == ora.inner_iters and (r.winner == ora.winner).all()
        print(seed, "ok" if ok else "MISMATCH", r.stats["inner_iters"], ora.inner_iters, r.stats["inc_valuations"], flush=True)
    except PGError as e:
        print(seed, "ERR", e, flush=True)
