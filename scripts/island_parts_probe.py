"""Island-throughput leg split into its parts (seeding, session, runs,
migration, results); `after-evolve` first runs the time-to-converge GA."""
import sys, time
sys.path.insert(0, ".")
import torch, numpy as np
from paper_2206_01288_b200 import PAPER_WORKLOAD, scenario_case
from paper_2206_01288_b200 import scheduler as S
g = scenario_case(5).graph(); w = PAPER_WORKLOAD
I = 1184
if len(sys.argv) > 1 and sys.argv[1] == "after-evolve":
    t = time.perf_counter(); S.evolve(g, w, S.ScheduleConfig(pop_size=64, generations=1000, local_search="ours", seed=0)); torch.cuda.synchronize(); print(f"evolve {time.perf_counter() - t:.3f}")
for rep in range(2):
    cfg = S.ScheduleConfig(pop_size=64, generations=100, local_search="ours", seed=1)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    rngs = S.island_seeds(cfg.seed, I, offset=0); t1 = time.perf_counter()
    sess = S.GASession(g, w, cfg, rngs, mode="warp"); torch.cuda.synchronize(); t2 = time.perf_counter()
    src = S.migration_sources(0, 1, I)
    tr = 0; tm = 0
    for gen in (25, 50, 75, 100):
        a = time.perf_counter(); sess.run(gen); torch.cuda.synchronize(); tr += time.perf_counter() - a
        if gen < 100:
            a = time.perf_counter(); gr, co = sess.export_elites(2); sess.import_elites(gr, co, src); torch.cuda.synchronize(); tm += time.perf_counter() - a
    a = time.perf_counter(); res = sess.results([cfg.seed] * I); t3 = time.perf_counter()
    print(f"seeds {t1-t0:.3f} session {t2-t1:.3f} runs {tr:.3f} migrate {tm:.3f} results {t3-a:.3f} total {t3-t0:.3f}")
import gc
for rep in range(4):
    cfg = S.ScheduleConfig(pop_size=64, generations=100, local_search="ours", seed=1)
    if rep >= 2:
        gc.collect()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = S.evolve_islands(g, w, cfg, I, migrate_every=25, elites=2)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    del r
    print(f"evolve_islands {t1 - t0:.3f} (gc.collect before: {rep >= 2})")
