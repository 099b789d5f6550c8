"""Config-4 pricing probe (512 devices, 16 x 32): device-resident evals/s of
the CTA Held-Karp path; used for ncu captures of eval_cta_kernel."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2206_01288_b200 import _native as N
from paper_2206_01288_b200.netmodel import config4_scenario
from paper_2206_01288_b200.workload import WorkloadSpec

P = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
g = config4_scenario().graph()
w = WorkloadSpec(16, 32, 268_435_456, 201_326_592)
dev = torch.device("cuda:0")
inst = N.instance_for(g, w, 0)
x = torch.sort(torch.argsort(torch.rand((P, 512), device=dev), dim=1).to(torch.int16).view(P, 16, 32), dim=2).values.contiguous()
o = [torch.empty(P, dtype=torch.float64, device=dev) for _ in range(3)]
sp = torch.cuda.current_stream(dev).cuda_stream
def call():
    N.check(N.lib().hs_eval_batch_ex(inst.handle, x.data_ptr(), P, o[0].data_ptr(), o[1].data_ptr(), o[2].data_ptr(),
                                     None, None, None, 0, sp), "eval")
call(); torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(reps): call()
torch.cuda.synchronize()
print(f"config4 16x32: {P * reps / (time.perf_counter() - t0):.1f} evals/s, total[0] {o[0][0].item()!r}")
