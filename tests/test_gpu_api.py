"""GPU parity of the single-call public surface: bottleneck_perfect_matching,
coarsen, datap_cost_group and the exhaustive k! oracles, bitwise against
vectors the reference produced (tests/golden/solvers.json, api.json)."""
from __future__ import annotations

import json

import numpy as np
import pytest

from tests import _instances as I
from tests._instances import fx

pytestmark = pytest.mark.gpu

hs = pytest.importorskip("paper_2206_01288_b200")
API = json.loads((I.GOLDEN / "api.json").read_text())
SOLVERS = json.loads((I.GOLDEN / "solvers.json").read_text())


def _mat(rec, key):
    k = rec.get("k", rec.get("m"))
    return np.array([fx(x) for x in rec[key]]).reshape(k, k)


def test_bottleneck_perfect_matching_golden():
    from paper_2206_01288_b200.combinatorics import bottleneck_matchings, bottleneck_perfect_matching
    for rec in SOLVERS["matching"]:
        w = _mat(rec, "w")
        r = bottleneck_perfect_matching(w)
        assert r.bottleneck == fx(rec["value"])
        assert list(r.pairs) == rec["pairs"]
    # batched, mixed values, one launch
    recs = [r for r in SOLVERS["matching"] if r["m"] == 8]
    vals, pairs = bottleneck_matchings(np.stack([_mat(r, "w") for r in recs]))
    assert [fx(r["value"]) for r in recs] == vals.tolist()
    assert [r["pairs"] for r in recs] == pairs.tolist()


@pytest.mark.parametrize("kind", ["brute_matching", "brute_tsp"])
def test_brute_force_oracles(kind):
    from paper_2206_01288_b200 import combinatorics as Cb
    for rec in API[kind]:
        w = _mat(rec, "w")
        if kind == "brute_matching":
            r = Cb.brute_force_bottleneck_matching(w)
            assert (list(r.pairs), r.bottleneck) == (rec["pairs"], fx(rec["value"]))
        else:
            r = Cb.brute_force_open_loop_tsp(w)
            assert (list(r.order), r.total) == (rec["order"], fx(rec["total"]))
    with pytest.raises(ValueError, match="limited to k <= 10"):
        Cb.brute_force_open_loop_tsp(np.zeros((11, 11)))


def test_coarsen_golden():
    for rec in API["coarsen"]:
        g, w = I.instance(rec["instance"])
        p = hs.Partition.from_groups(rec["groups"])
        cg = hs.coarsen(g, p, w)
        assert cg.k == w.d_pp
        assert cg.edge_cost.ravel().tolist() == [fx(x) for x in rec["edge"]]
        got = [[j, j2, list(r.pairs), r.bottleneck] for (j, j2), r in sorted(cg.matchings.items())]
        assert got == [[j, j2, pr, fx(v)] for j, j2, pr, v in rec["matchings"]]
        # pipeline_cost over the coarsened graph equals comm_cost's pipeline level
        assert hs.pipeline_cost(cg)[0] == hs.comm_cost(g, p, w).pipelinep


def test_datap_cost_group_golden():
    for rec in API["datap_group"]:
        g, w = I.instance(rec["instance"])
        assert hs.datap_cost_group(g, rec["group"], w) == fx(rec["value"])
    g, w = I.instance("case5")
    with pytest.raises(hs.CostModelError, match="duplicate device"):
        hs.datap_cost_group(g, [0, 0, 1, 2, 3, 4, 5, 6], w)
    with pytest.raises(hs.CostModelError, match="does not match d_dp"):
        hs.datap_cost_group(g, [0, 1], w)


@pytest.mark.parametrize("name", ["case5", "config1", "r10_10x1", "config5"])
def test_datap_cost_is_the_data_parallel_level_only(name):
    """datap_cost == comm_cost's datap / per_group where exact pricing exists,
    and needs no Held-Karp (works for any d_pp, like costmodel.py:171-175)."""
    from oracle import oracle as O
    g, w = I.instance(name)
    rng = np.random.default_rng(3)
    for _ in range(3):
        p = hs.random_partition(rng, g.lat.shape[0], w.d_pp, w.d_dp)
        mx, per = hs.datap_cost(g, p, w)
        if w.d_pp <= 16:
            cb = hs.comm_cost(g, p, w)
            assert mx == cb.datap and per == cb.per_group_datap
        _, d, _ = O.Oracle.of(g, w).comm_cost_batch(np.asarray([p.groups], dtype=np.int16)) if w.d_pp <= 16 \
            else (None, [mx], None)
        assert mx == d[0] and mx == max(per)
