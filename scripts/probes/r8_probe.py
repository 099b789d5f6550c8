import sys, os
sys.path.insert(0, "/root/repo")
from tests import _instances as I
from paper_2206_01288_b200 import scheduler as S
g, w = I.instance("r8_4x2")
cfg = S.ScheduleConfig(pop_size=8, generations=40, local_search=sys.argv[1], seed=0)
try:
    r = S.evolve(g, w, cfg)
    print("ok", r.best_cost.total)
except Exception as e:
    print("ERR", e)
