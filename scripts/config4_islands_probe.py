"""Config 4 island model on one GPU: time per phase (HS_GA_PROFILE=1 prints
island 0's driver cycle counters), batch-priced vs in-kernel pricing
(HS_GA_BATCH=0)."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2206_01288_b200 import scheduler as S  # noqa: E402
from paper_2206_01288_b200.netmodel import config4_scenario  # noqa: E402
from paper_2206_01288_b200.workload import WorkloadSpec  # noqa: E402

g4 = config4_scenario().graph()
w4 = WorkloadSpec(16, 32, 268_435_456, 201_326_592)
gens = int(sys.argv[1]) if len(sys.argv) > 1 else 3
islands = int(sys.argv[2]) if len(sys.argv) > 2 else 148
cfg = S.ScheduleConfig(pop_size=16, generations=gens, local_search="ours", seed=5)
sess = S.GASession(g4, w4, cfg, S.island_seeds(cfg.seed, islands))
torch.cuda.synchronize()
t0 = time.perf_counter()
sess.run(1)
torch.cuda.synchronize()
t1 = time.perf_counter()
sess.run(gens)
torch.cuda.synchronize()
t2 = time.perf_counter()
res = sess.results()
t3 = time.perf_counter()
ev = sum(r.evaluations for r in res)
print(f"islands {islands}: init+gen1 {t1 - t0:.3f} s, gens 2..{gens} {t2 - t1:.3f} s, results/finalize {t3 - t2:.3f} s, "
      f"{islands * gens / (t3 - t0):.1f} island-gens/s, {ev} evaluations")
