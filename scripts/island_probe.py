"""Island throughput: CTA-per-island vs warp-per-island (case 5, ours)."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2206_01288_b200 import PAPER_WORKLOAD, scenario_case
from paper_2206_01288_b200 import scheduler as S
g = scenario_case(5).graph()
gens = int(sys.argv[1]) if len(sys.argv) > 1 else 50
sms = torch.cuda.get_device_properties(0).multi_processor_count
for mode, I in (("cta", sms), ("warp", sms * 8)):
    cfg = S.ScheduleConfig(pop_size=64, generations=gens, local_search="ours", seed=1)
    sess = S.GASession(g, PAPER_WORKLOAD, cfg, S.island_seeds(1, I), mode=mode)
    torch.cuda.synchronize()
    t = time.perf_counter()
    sess.run(gens)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"{mode}: {I} islands x {gens} gens in {dt:.3f} s -> {I * gens / dt:.0f} island-generations/s")
