"""GPU exhaustive search (brute_force_best, costmodel.py:232-266)."""
from __future__ import annotations

from itertools import combinations

import numpy as np
import pytest

from oracle import oracle as O
from tests import _instances as I

pytestmark = pytest.mark.gpu

hs = pytest.importorskip("paper_2206_01288_b200")


def enumerate_partitions(devices, m):
    """Independent restatement of the reference enumeration order."""
    if not devices:
        yield ()
        return
    head, rest = devices[0], devices[1:]
    for partners in combinations(rest, m - 1):
        taken = set(partners)
        remaining = tuple(d for d in rest if d not in taken)
        for tail in enumerate_partitions(remaining, m):
            yield ((head,) + partners,) + tail


@pytest.mark.parametrize("n,k,m", [(8, 4, 2), (8, 2, 4), (6, 3, 2), (12, 3, 4), (9, 3, 3)])
def test_unrank_matches_reference_enumeration_order(n, k, m):
    import torch
    from paper_2206_01288_b200 import _native as N
    want = np.array(list(enumerate_partitions(tuple(range(n)), m)), dtype=np.int16)
    assert N.lib().hs_count_partitions(n, m) == len(want)
    out = torch.empty((len(want), k, m), dtype=torch.int16, device="cuda")
    N.check(N.lib().hs_unrank_partitions(n, k, m, 0, len(want), out.data_ptr(), None), "unrank")
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), want)


def test_g4_optimum_and_reference_limit():
    g, w = I.instance("g4")
    p, cb = hs.brute_force_best(g, w)
    assert p == hs.Partition(((0, 1), (2, 3))) and cb.total == pytest.approx(2.502, rel=1e-9)
    g10 = I.homogeneous(10)
    with pytest.raises(hs.CostModelError, match="limited to 8"):
        hs.brute_force_best(g10, hs.WorkloadSpec(5, 2, 1.0, 1.0))


def test_homogeneous_tie_is_lexicographically_smallest():
    g = I.homogeneous(4)
    p, _ = hs.brute_force_best(g, hs.WorkloadSpec(2, 2, 1.0, 1.0))
    assert p == hs.Partition(((0, 1), (2, 3)))


@pytest.mark.parametrize("name,max_dev", [("r8_4x2", 8), ("r8_2x4", 8), ("r12_3x4", 12), ("r12_4x3", 12)])
def test_brute_force_vs_oracle(name, max_dev):
    g, w = I.instance(name)
    p, cb = hs.brute_force_best(g, w, max_devices=max_dev)
    parts = np.array(list(enumerate_partitions(tuple(range(g.n)), w.d_dp)), dtype=np.int16)
    t, _, _ = O.Oracle.of(g, w).comm_cost_batch(parts, threads=O.cpu_count())
    i = int(np.argmin(t))
    assert [list(x) for x in p.groups] == parts[i].tolist() and cb.total == t[i]


@pytest.mark.parametrize("name", ["r16_4x4", "r16_2x8"])
def test_brute_force_n16_optimum_properties(name):
    """N = 16 (2.6M balanced 4x4 partitions; §8(f) row 2 asks for 12-16):
    the oracle re-prices the returned optimum to the same bits, and no
    partition in a 20k random sample (priced by the oracle) is cheaper."""
    g, w = I.instance(name)
    p, cb = hs.brute_force_best(g, w, max_devices=16)
    orc = O.Oracle.of(g, w)
    t, _, _ = orc.comm_cost_batch(np.asarray([p.groups], dtype=np.int16))
    assert t[0] == cb.total
    rng = np.random.default_rng(16)
    sample = np.sort(rng.permuted(np.tile(np.arange(16, dtype=np.int16), (20_000, 1)), axis=1)
                     .reshape(-1, w.d_pp, w.d_dp), axis=2)
    ts, _, _ = orc.comm_cost_batch(sample, threads=O.cpu_count())
    assert ts.min() >= cb.total
