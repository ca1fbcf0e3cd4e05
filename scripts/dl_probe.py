import os,sys
sys.path.insert(0,'/root/repo')
os.environ["PGSI_SMALL_MAX"]="0"
import pg_inputs as gi
from paper_1705_02313_b200 import Game
g=gi.random_game(50000,8,2,5,1)
try:
    r=Game.from_game(g).solve()
    print(r.stats["device_loop_solves"], r.stats["inner_iters"])
except Exception as e:
    print("ERR", e)
