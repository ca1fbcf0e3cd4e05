import os,sys
sys.path.insert(0,'/root/repo')
os.environ.setdefault("PGSI_SMALL_MAX","0"); os.environ.setdefault("PGSI_CLUSTER","0"); os.environ.setdefault("PGSI_DEVICE_LOOP","2")
import pg_inputs as gi
from paper_1705_02313_b200 import Game
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
g=gi.random_game(n,8,2,5,1)
print("solving", n, {k: os.environ.get(k) for k in ("PGSI_INC_EVEN","PGSI_DEVICE_LOOP")}, flush=True)
r=Game.from_game(g).solve()
print("ok", r.stats["device_loop_solves"], r.stats["inner_iters"], r.stats["outer_passes"], r.stats["inc_even_switches"], flush=True)
