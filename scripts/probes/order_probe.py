"""Device-resident evals/s with the full CostBreakdown (per-group + stage
order) at N = 64, 8x8, case 5, P = 2^20."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2206_01288_b200 import _native as N  # noqa: E402
from paper_2206_01288_b200 import PAPER_WORKLOAD, scenario_case  # noqa: E402

P = 1 << 20
g = scenario_case(5).graph()
inst = N.instance_for(g, PAPER_WORKLOAD, 0)
gen = torch.Generator(device="cuda")
gen.manual_seed(3)
x = torch.sort(torch.argsort(torch.rand((P, 64), device="cuda", generator=gen), dim=1).to(torch.int16).view(P, 8, 8),
               dim=2).values.contiguous()
o = [torch.empty(P, dtype=torch.float64, device="cuda") for _ in range(3)]
pg = torch.empty((P, 8), dtype=torch.float64, device="cuda")
od = torch.empty((P, 8), dtype=torch.int8, device="cuda")
bad = torch.zeros(1, dtype=torch.int32, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
for order in (False, True):
    def call():
        N.check(N.lib().hs_eval_batch(inst.handle, x.data_ptr(), P, o[0].data_ptr(), o[1].data_ptr(), o[2].data_ptr(),
                                      pg.data_ptr(), od.data_ptr() if order else None, bad.data_ptr(), sp), "eval")
    call()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        call()
    b.record()
    torch.cuda.synchronize()
    print(f"per_group{' + order' if order else ''}: {P * 5 / (a.elapsed_time(b) / 1e3):.3e} evals/s")
