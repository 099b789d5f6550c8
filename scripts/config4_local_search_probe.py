"""hs_local_search on B config-4 partitions (512 devices, 16 x 32, ours):
batch-priced snapshots vs in-kernel pricing (HS_GA_BATCH=0 in the env)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2206_01288_b200 import _native as N  # noqa: E402
from paper_2206_01288_b200 import scheduler as S  # noqa: E402
from paper_2206_01288_b200.netmodel import config4_scenario  # noqa: E402
from paper_2206_01288_b200.workload import WorkloadSpec  # noqa: E402

g = config4_scenario().graph()
w = WorkloadSpec(16, 32, 268_435_456, 201_326_592)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 148
rng = np.random.default_rng(8)
parts = np.stack([np.array(S.random_partition(rng, g.n, w.d_pp, w.d_dp).groups, dtype=np.int16) for _ in range(B)])
inst = N.instance_for(g, w)
out = np.empty_like(parts)
ev = np.empty(B, dtype=np.int32)
ts = []
for rep in range(3):
    st = S._states([np.random.default_rng(300 + i) for i in range(B)])
    t0 = time.perf_counter()
    N.check(N.lib().hs_local_search(inst.handle, 0, 8, B, parts.ctypes.data, st, out.ctypes.data, None,
                                    ev.ctypes.data), "hs_local_search")
    ts.append(time.perf_counter() - t0)
t = float(np.median(ts))
print(f"local_search, {B} config-4 partitions: {t:.3f} s ({B / t:.1f} partitions/s, {int(ev.sum())} snapshots priced)")
