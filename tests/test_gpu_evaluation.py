"""GPU parity of the fixed-layout path (evaluation.py) and the pinned
case-5 regression of the reference acceptance suite (criterion 6)."""
from __future__ import annotations

import json

import numpy as np
import pytest

from oracle import oracle as O
from tests import _instances as I
from tests._instances import fx

pytestmark = pytest.mark.gpu

hs = pytest.importorskip("paper_2206_01288_b200")
from paper_2206_01288_b200 import evaluation as E  # noqa: E402
from paper_2206_01288_b200 import scheduler as S  # noqa: E402

PINNED_CASE5_RATIO = 0.22732911104944017  # reference tests/test_acceptance.py:49


def test_materialize_and_evaluate_match_golden():
    for c in I.fixture("assignments.json")["materialize"]:
        g, w = I.instance(c["inst"])
        a = E.materialize(g, hs.Partition.from_groups(c["groups"]), w)
        assert [list(r) for r in a.grid] == c["grid"] and list(a.order) == c["order"]
        cb = E.evaluate_assignment(g, a, w)
        assert cb.total == fx(c["total"]) and cb.datap == fx(c["datap"]) and cb.pipelinep == fx(c["pipelinep"])


def test_random_assignments_match_golden():
    for c in I.fixture("assignments.json")["random"]:
        g, w = I.instance(c["inst"])
        rng = np.random.Generator(np.random.PCG64(0))
        s = rng.bit_generator.state
        s["state"]["state"], s["state"]["inc"] = int(c["state0"][0]), int(c["state0"][1])
        s["has_uint32"], s["uinteger"] = 0, 0
        rng.bit_generator.state = s
        a = E.random_assignment(rng, g.n, w.d_pp, w.d_dp)
        assert [list(r) for r in a.grid] == c["grid"] and list(a.order) == c["order"]
        assert E.evaluate_assignment(g, a, w).total == fx(c["total"])


@pytest.mark.parametrize("case", [1, 2, 3, 4, 5])
def test_evaluate_materialize_identity_bitwise(case):
    """Acceptance criterion 5 at scale: evaluate(materialize(p)) == comm_cost(p)."""
    g, w = I.instance(f"case{case}")
    rng = np.random.default_rng(case)
    parts = np.sort(rng.permuted(np.tile(np.arange(64, dtype=np.int16), (2000, 1)), axis=1).reshape(-1, 8, 8), axis=2)
    grids, _ = E.materialize_batch(g, parts, w)
    via = E.evaluate_assignments(g, grids, w)
    direct = hs.comm_cost_batch(g, parts, w)
    for key in ("total", "datap", "pipelinep"):
        assert np.array_equal(via[key], direct[key])
    orc = O.Oracle.of(g, w)
    for i in range(20):
        og, oo = orc.materialize(parts[i].astype(np.int32))
        assert og.tolist() == grids[i].tolist()


def test_pinned_case5_ratio_reproduced_exactly():
    """Criterion 6: 1000-generation GA vs 100 seeded random layouts on case 5."""
    g, w = I.instance("case5")
    res = S.evolve(g, w, S.ScheduleConfig(pop_size=64, generations=1000, local_search="ours", seed=0))
    totals = E.random_totals(g, w, 0, 100)
    ratio = res.best_cost.total / float(np.mean(totals))
    assert ratio == PINNED_CASE5_RATIO


def test_compare_baselines_report():
    g, w = I.instance("g4")
    rep = E.compare_baselines(g, w, S.ScheduleConfig(pop_size=8, generations=10, seed=0), random_trials=5)
    d = rep.to_dict()
    assert d["random"]["count"] == 5 and len(d["random"]["totals"]) == 5
    assert rep.speedup_vs_mean_random == rep.random_mean / rep.scheduled.total
    with pytest.raises(E.AssignmentError):
        E.compare_baselines(g, w, S.ScheduleConfig(pop_size=8, generations=10), random_trials=0)
