"""BASELINE config 5 (1024 devices): heuristic stage ordering for d_pp > 16
and the gains-only local-search stress at 32 x 32, vs the reference's own
outputs (tests/golden/big.json) and the oracle."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from tests import _instances as I
from tests._instances import fx

pytestmark = pytest.mark.gpu

hs = pytest.importorskip("paper_2206_01288_b200")
from paper_2206_01288_b200 import scheduler as S  # noqa: E402
from paper_2206_01288_b200.netmodel import random_graph  # noqa: E402

C5B = hs.WorkloadSpec(32, 32, 268_435_456, 201_326_592)


@pytest.fixture(scope="module")
def g1024():
    return random_graph(0, 1024)


def test_heuristic_paths_vs_golden_and_oracle():
    for c in I.fixture("solvers.json")["tsp_heuristic"]:
        k = c["k"]
        w = np.array([fx(x) for x in c["w"]]).reshape(k, k)
        r = hs.open_loop_tsp(w, heuristic=True)
        assert r.total == fx(c["total"]) and list(r.order) == c["order"]
    rng = np.random.default_rng(3)
    for k in (17, 24, 32, 48, 64):
        for _ in range(3):
            w = rng.uniform(1, 10, size=(k, k))
            w = (w + w.T) / 2.0
            np.fill_diagonal(w, 0.0)
            r = hs.open_loop_tsp(w, heuristic=True)
            o, t = O.open_loop_tsp(w, heuristic=True)
            assert r.total == t and tuple(r.order) == o


def test_exact_pricing_refuses_more_than_16_stages(g1024):
    p = S.random_partition(np.random.default_rng(0), 1024, 32, 32)
    with pytest.raises(ValueError, match="heuristic=True"):
        hs.comm_cost(g1024, p, C5B)


def test_config5_heuristic_costs_vs_reference(g1024):
    for c in I.fixture("big.json")["heuristic_costs"]:
        cb = hs.comm_cost(g1024, hs.Partition.from_groups(c["groups"]), C5B, heuristic=True)
        assert cb.total == fx(c["total"]) and cb.datap == fx(c["datap"]) and cb.pipelinep == fx(c["pipelinep"])
        assert list(cb.pipeline_order.order) == c["order"]


def test_config5_heuristic_batch_vs_oracle(g1024):
    rng = np.random.default_rng(8)
    parts = np.stack([np.sort(rng.permutation(1024).reshape(32, 32), axis=1) for _ in range(6)]).astype(np.int16)
    r = hs.comm_cost_batch(g1024, parts, C5B, heuristic=True, order=True)
    orc = O.Oracle.of(g1024, C5B)
    for i in range(len(parts)):
        t, d, p, order = orc.comm_cost_heuristic(parts[i])
        assert r["total"][i] == t and r["datap"][i] == d and r["pipelinep"][i] == p
        assert list(r["order"][i]) == list(order)


def test_config5_gains_only_passes_vs_reference(g1024):
    for c in I.fixture("big.json")["passes"]:
        rng = np.random.Generator(np.random.PCG64(c["seed"]))
        ch, out = S.refine_pass(g1024, C5B, hs.Partition.from_groups(c["groups"]), c["kind"], rng, c["phase"])
        assert ch == c["changed"]
        assert [list(x) for x in out.groups] == [sorted(x) for x in c["out"]]
        st = rng.bit_generator.state
        assert [str(st["state"]["state"]), st["has_uint32"], st["uinteger"]] == c["rng_after"]
