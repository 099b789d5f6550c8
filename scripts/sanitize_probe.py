"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck):
every hot kernel family once, tiny sizes, results checked against the C
oracle so a clean sanitizer log is also a correct run.

    compute-sanitizer --tool memcheck python scripts/sanitize_probe.py
"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2206_01288_b200 import PAPER_WORKLOAD, comm_cost_batch, scenario_case  # noqa: E402
from paper_2206_01288_b200 import scheduler as S  # noqa: E402
from paper_2206_01288_b200.netmodel import config4_scenario  # noqa: E402
from paper_2206_01288_b200.workload import WorkloadSpec  # noqa: E402


def parts(seed, P, n, k, m):
    rng = np.random.default_rng(seed)
    return np.sort(rng.permuted(np.tile(np.arange(n, dtype=np.int16), (P, 1)), axis=1).reshape(P, k, m), axis=2)


def check(name, got, want):
    assert np.array_equal(got, want), name
    print(f"ok {name}", flush=True)


g5, w5 = scenario_case(5).graph(), PAPER_WORKLOAD
x = parts(1, 300, 64, 8, 8)
want = O.Oracle.of(g5, w5).comm_cost_batch(x)[0]
check("eval8 (k=8, no order)", comm_cost_batch(g5, x, w5)["total"], want)
check("eval_warp (k=8, order)", comm_cost_batch(g5, x, w5, order=True)["total"], want)
g4, w4 = config4_scenario().graph(), WorkloadSpec(16, 32, 268_435_456, 201_326_592)
x4 = parts(2, 3, 512, 16, 32)
want4 = O.Oracle.of(g4, w4).comm_cost_batch(x4)[0]
check("stage + hk_cluster (k=16)", comm_cost_batch(g4, x4, w4)["total"], want4)
check("eval_cta (k=16, order)", comm_cost_batch(g4, x4, w4, order=True)["total"], want4)
cfg = S.ScheduleConfig(pop_size=16, generations=4, local_search="ours", seed=3)
r = S.evolve(g5, w5, cfg)  # CTA island: sweep waves over 8 warps + register chains
o = O.Oracle.of(g5, w5).evolve(16, 4, "ours", seed=3)
check("ga_kernel cta island (sweep waves, chains)", np.array([r.best_cost.total]), np.array([o["total"]]))
sess = S.GASession(g5, w5, cfg, S.island_seeds(3, 9), mode="warp")
sess.run(cfg.generations)
print(f"ok ga_kernel warp islands: {len(sess.results())} islands", flush=True)
cfgk = S.ScheduleConfig(pop_size=8, generations=2, local_search="kl", seed=5)
r = S.evolve(g5, w5, cfgk)
o = O.Oracle.of(g5, w5).evolve(8, 2, "kl", seed=5)
check("ga_kernel kl", np.array([r.best_cost.total]), np.array([o["total"]]))
print("sanitize probe done")
