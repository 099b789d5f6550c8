"""BASELINE config 5 local-search stress: one refinement pass (ours sweep /
ours chains / KL, gains only) over 1,024 partitions of 1,024 devices in
32 x 32 groups (hs_refine_pass); median of 5 calls after a warm-up."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2206_01288_b200 import _native as N  # noqa: E402
from paper_2206_01288_b200 import scheduler as S  # noqa: E402
from paper_2206_01288_b200.netmodel import random_graph  # noqa: E402
from paper_2206_01288_b200.workload import WorkloadSpec  # noqa: E402

g5 = random_graph(0, 1024)
w5 = WorkloadSpec(32, 32, 1 << 30, 3 << 26)
inst = N.instance_for(g5, w5, 0)
B = 1024
rng = np.random.default_rng(0)
parts = np.stack([np.sort(rng.permutation(1024).reshape(32, 32), axis=1) for _ in range(B)]).astype(np.int16)
res = np.empty_like(parts)
ch = np.zeros(B, dtype=np.int32)
for name, kind, phase in (("ours_sweep", 0, 0), ("ours_chains", 0, 1), ("kl", 1, 0)):
    ts = []
    for rep in range(6):
        st = S._states([np.random.default_rng(i) for i in range(B)])
        t0 = time.perf_counter()
        N.check(N.lib().hs_refine_pass(inst.handle, kind, phase, B, parts.ctypes.data, st, res.ctypes.data,
                                       ch.ctypes.data), "hs_refine_pass")
        ts.append(time.perf_counter() - t0)
    t = float(np.median(ts[1:]))
    print(f"{name}: {B / t:.0f} passes/s ({t * 1e3:.1f} ms per {B}), changed {int(ch.sum())}")
