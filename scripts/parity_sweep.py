"""Bitwise parity at scale: comm_cost_batch (GPU, host-buffer path) against
the C oracle on 1M random layouts per paper scenario plus configs 1 and 4
(the oracle is the test-infrastructure restatement of costmodel.py, pinned
to the reference's own outputs by tests/test_oracle_golden.py).

    python scripts/parity_sweep.py [layouts_per_case]
"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2206_01288_b200 import costmodel as C  # noqa: E402
from tests import _instances as I  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20


def parts(seed, count, n, k, m):
    rng = np.random.default_rng(seed)
    out = np.empty((count, k, m), dtype=np.int16)
    for lo in range(0, count, 1 << 16):
        hi = min(count, lo + (1 << 16))
        out[lo:hi] = np.sort(rng.permuted(np.tile(np.arange(n, dtype=np.int16), (hi - lo, 1)), axis=1)
                             .reshape(hi - lo, k, m), axis=2)
    return out


total = 0
for name, count in [(f"case{c}", N) for c in range(1, 6)] + [("config1", N), ("config4", 2048)]:
    g, w = I.instance(name)
    p = parts(hash(name) % 1000, count, g.lat.shape[0], w.d_pp, w.d_dp)
    t0 = time.perf_counter()
    r = C.comm_cost_batch(g, p, w)
    t_gpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    t, d, pp = O.Oracle.of(g, w).comm_cost_batch(p, threads=O.cpu_count())
    t_cpu = time.perf_counter() - t0
    ok = np.array_equal(r["total"], t) and np.array_equal(r["datap"], d) and np.array_equal(r["pipelinep"], pp)
    total += count
    print(f"{name}: {count} layouts ({w.d_pp}x{w.d_dp}, n={g.lat.shape[0]}): bitwise {'EQUAL' if ok else 'DIFFERENT'}"
          f" (GPU {t_gpu:.2f} s incl. copies, oracle {t_cpu:.1f} s on {O.cpu_count()} threads)", flush=True)
    assert ok, name
print(f"all {total} layouts bit-identical to the oracle")
