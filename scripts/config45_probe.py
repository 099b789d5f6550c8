"""Device-resident evals/s on BASELINE configs 4 and 5 (hs_eval_batch_ex),
for A/B runs of the d_pp 9..16 kernels (HS_LIB_PATH selects a variant)."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2206_01288_b200 import _native as N  # noqa: E402
from paper_2206_01288_b200.netmodel import config4_scenario, random_graph  # noqa: E402
from paper_2206_01288_b200.workload import WorkloadSpec  # noqa: E402

P4 = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
gen = torch.Generator(device="cuda")
gen.manual_seed(77)


def rate(g, w, P, reps=2):
    n = g.lat.shape[0]
    x = torch.sort(torch.argsort(torch.rand((P, n), device="cuda", generator=gen), dim=1).to(torch.int16)
                   .view(P, w.d_pp, w.d_dp), dim=2).values.contiguous()
    inst = N.instance_for(g, w, 0)
    o = [torch.empty(P, dtype=torch.float64, device="cuda") for _ in range(3)]
    sp = torch.cuda.current_stream().cuda_stream

    def call():
        N.check(N.lib().hs_eval_batch_ex(inst.handle, x.data_ptr(), P, o[0].data_ptr(), o[1].data_ptr(),
                                         o[2].data_ptr(), None, None, None, 0, sp), "hs_eval_batch_ex")
    call()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        call()
    torch.cuda.synchronize()
    return P * reps / (time.perf_counter() - t), float(o[0][:8].sum())


print("config4 16x32 P=%d: %.0f evals/s (checksum %r)" % ((P4,) + rate(config4_scenario().graph(),
                                                                       WorkloadSpec(16, 32, 268_435_456, 201_326_592),
                                                                       P4)))
print("config5 16x64 P=2048: %.0f evals/s (checksum %r)" % rate(random_graph(0, 1024),
                                                               WorkloadSpec(16, 64, 1 << 30, 3 << 26), 2048))
