"""Config 5 pricing (1024 devices, 16 x 64, random graph): evals/s at P."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2206_01288_b200 import _native as N  # noqa: E402
from paper_2206_01288_b200.netmodel import random_graph  # noqa: E402
from paper_2206_01288_b200.workload import WorkloadSpec  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
g, w = random_graph(0, 1024), WorkloadSpec(16, 64, 1 << 30, 3 << 26)
inst = N.instance_for(g, w, 0)
gen = torch.Generator(device="cuda")
gen.manual_seed(5)
x = torch.sort(torch.argsort(torch.rand((P, 1024), device="cuda", generator=gen), dim=1).to(torch.int16)
               .view(P, 16, 64), dim=2).values.contiguous()
o = [torch.empty(P, dtype=torch.float64, device="cuda") for _ in range(3)]
sp = torch.cuda.current_stream().cuda_stream
call = lambda: N.check(N.lib().hs_eval_batch_ex(inst.handle, x.data_ptr(), P, o[0].data_ptr(), o[1].data_ptr(),  # noqa
                                                o[2].data_ptr(), None, None, None, 0, sp), "eval")
call()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
call()
b.record()
torch.cuda.synchronize()
print(f"config 5 16x64 P={P}: {P / (a.elapsed_time(b) / 1e3):.0f} evals/s")
