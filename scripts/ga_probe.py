"""Small GA run used for profiling the K3 kernel (one island, case 5)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2206_01288_b200 import PAPER_WORKLOAD, scenario_case
from paper_2206_01288_b200 import scheduler as S
gens = int(sys.argv[1]) if len(sys.argv) > 1 else 50
kind = sys.argv[2] if len(sys.argv) > 2 else "ours"
g = scenario_case(5).graph()
cfg = S.ScheduleConfig(pop_size=64, generations=gens, local_search=kind, seed=0)
S.evolve(g, PAPER_WORKLOAD, S.ScheduleConfig(pop_size=8, generations=2, local_search=kind))
torch.cuda.synchronize()
t = time.perf_counter()
r = S.evolve(g, PAPER_WORKLOAD, cfg)
torch.cuda.synchronize()
print(f"{kind} {gens} gens: {time.perf_counter() - t:.3f} s, best {r.best_cost.total}, evals {r.evaluations}")
