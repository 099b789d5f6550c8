"""Pin the CPU oracle (oracle/) against golden vectors from the reference.

CPU-only.  The fixtures under tests/golden/ were produced by running the
reference itself (tests/golden/make_golden.py); the oracle must reproduce
them bit for bit before it may serve as the checker for the GPU path.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from tests import _instances as I
from tests._instances import fx


def test_instances_reproduce_reference_matrices():
    for name, m in I.meta().items():
        g, w = I.instance(name)
        assert I.sha(g.lat) == m["lat_sha"], name
        assert I.sha(g.bw) == m["bw_sha"], name


def test_oracle_tables_match_reference_surrogate():
    for name, m in I.meta().items():
        g, w = I.instance(name)
        _, _, sw = O.Oracle.of(g, w).tables()
        assert I.sha(sw) == m["sw_sha"], name


@pytest.mark.parametrize("name", sorted(I.meta()))
def test_oracle_comm_cost_bitwise(name):
    g, w = I.instance(name)
    orc = O.Oracle.of(g, w)
    C = I.costs()
    parts = C[f"{name}/parts"]
    for i in range(parts.shape[0]):
        t, d, p, pg, order = orc.comm_cost(parts[i])
        assert t == C[f"{name}/total"][i]
        assert d == C[f"{name}/datap"][i]
        assert p == C[f"{name}/pipelinep"][i]
        assert np.array_equal(pg, C[f"{name}/per_group"][i])
        assert tuple(order) == tuple(C[f"{name}/order"][i])


def test_oracle_batch_threads_match_serial():
    g, w = I.instance("case5")
    orc = O.Oracle.of(g, w)
    parts = I.costs()["case5/parts"]
    t1, d1, p1 = orc.comm_cost_batch(parts, threads=1)
    t4, d4, p4 = orc.comm_cost_batch(parts, threads=4)
    assert np.array_equal(t1, t4) and np.array_equal(d1, d4) and np.array_equal(p1, p4)
    assert np.array_equal(t1, I.costs()["case5/total"])


def test_oracle_matching_and_tsp():
    fxs = I.fixture("solvers.json")
    for c in fxs["matching"]:
        m = c["m"]
        w = np.array([fx(x) for x in c["w"]]).reshape(m, m)
        assert O.bottleneck_value(w) == fx(c["value"])
        pairs, v = O.bottleneck_matching(w)
        assert v == fx(c["value"]) and list(pairs) == c["pairs"]
    for c in fxs["tsp"]:
        k = c["k"]
        w = np.array([fx(x) for x in c["w"]]).reshape(k, k)
        order, tot = O.open_loop_tsp(w)
        assert tot == fx(c["total"]) and list(order) == c["order"], k
    for c in fxs["tsp_heuristic"]:
        k = c["k"]
        w = np.array([fx(x) for x in c["w"]]).reshape(k, k)
        order, tot = O.open_loop_tsp(w, heuristic=True)
        assert tot == fx(c["total"]) and list(order) == c["order"], k


def _rng_after(st: O.PCG64State):
    return [str(st.as_tuple()[0]), st.as_tuple()[1], st.as_tuple()[2]]


def test_oracle_rng_primitives_match_numpy():
    for seed in range(60):
        g = np.random.Generator(np.random.PCG64(seed))
        st = O.PCG64State.from_generator(g)
        L = O.lib()
        import ctypes as C
        r = np.random.default_rng(seed + 7)
        for _ in range(30):
            op = int(r.integers(5))
            if op == 0:
                h = int(r.integers(1, 100))
                assert int(g.integers(h)) == L.orc_integers(C.byref(st), 0, h)
            elif op == 1:
                n = int(r.integers(0, 80))
                out = np.empty(max(n, 1), dtype=np.int32)
                L.orc_permutation(C.byref(st), n, out)
                assert list(g.permutation(n)) == list(out[:n])
            elif op == 2:
                n = int(r.integers(1, 50))
                s = int(r.integers(1, n + 1))
                out = np.empty(s, dtype=np.int32)
                L.orc_choice_noreplace_sorted(C.byref(st), n, s, out)
                assert sorted(int(x) for x in g.choice(n, size=s, replace=False)) == list(out)
            elif op == 3:
                lo = int(r.integers(0, 5))
                hi = lo + int(r.integers(1, 70))
                assert int(g.integers(lo, hi)) == L.orc_integers(C.byref(st), lo, hi)
            else:
                assert float(g.uniform(0.01, 0.25)) == L.orc_uniform(C.byref(st), 0.01, 0.25)
        gs = g.bit_generator.state
        assert st.as_tuple() == (gs["state"]["state"], gs["has_uint32"], gs["uinteger"])


def test_oracle_gains_and_fast_edge():
    fxs = I.fixture("search.json")
    for c in fxs["gains"]:
        g, w = I.instance(c["inst"])
        orc = O.Oracle.of(g, w)
        groups = np.array(c["groups"], dtype=np.int32)
        if c["kind"] == "ours":
            v = orc.gain_ours(groups, *c["args"])
        else:
            v = orc.gain_kl(groups, *c["args"])
        assert v == fx(c["value"])
    for c in fxs["fast_edge"]:
        g, w = I.instance(c["inst"])
        assert list(O.Oracle.of(g, w).fast_edge(c["grp"])) == c["edge"]


def test_oracle_passes():
    for c in I.fixture("search.json")["passes"]:
        g, w = I.instance(c["inst"])
        orc = O.Oracle.of(g, w)
        st = O.rng_state(c["seed"])
        ch, out = orc.one_pass(np.array(c["groups"], dtype=np.int32), c["kind"], st, c["phase"])
        assert ch == c["changed"], c["inst"]
        assert out.tolist() == c["out"], (c["inst"], c["kind"], c["phase"])
        assert _rng_after(st) == c["rng_after"]


def test_oracle_crossover():
    for c in I.fixture("search.json")["crossover"]:
        g, w = I.instance(c["inst"])
        st = O.rng_state(c["seed"])
        p1 = np.array(c["p1"], dtype=np.int32)
        p2 = np.array(c["p2"], dtype=np.int32)
        out = np.empty_like(p1)
        import ctypes as C
        O.lib().orc_crossover(p1, p2, w.d_pp, w.d_dp, C.byref(st), out)
        assert out.tolist() == c["child"]
        assert _rng_after(st) == c["rng_after"]


def test_oracle_local_search():
    for c in I.fixture("search.json")["local_search"]:
        g, w = I.instance(c["inst"])
        orc = O.Oracle.of(g, w)
        st = O.rng_state(np.random.default_rng(c["seed"]))
        out = orc.local_search(np.array(c["groups"], dtype=np.int32), c["kind"], st)
        assert out.tolist() == c["out"], (c["inst"], c["kind"])
        assert _rng_after(st) == c["rng_after"]


def _check_run(run):
    g, w = I.instance(run["inst"])
    res = O.Oracle.of(g, w).evolve(run["pop"], run["gens"], run["kind"], seed=run["seed"],
                                   patience=run["patience"])
    assert res["partition"].tolist() == run["partition"]
    assert res["total"] == fx(run["total"])
    assert res["datap"] == fx(run["datap"]) and res["pipelinep"] == fx(run["pipelinep"])
    assert [float(x) for x in res["per_group"]] == [fx(x) for x in run["per_group"]]
    assert list(res["order"]) == run["order"]
    assert res["evaluations"] == run["evaluations"]
    assert [float(x) for x in res["trace_best"]] == [fx(x) for x in run["trace_best"]]
    assert [float(x) for x in res["trace_mean"]] == [fx(x) for x in run["trace_mean"]]


@pytest.mark.parametrize("idx", range(len(I.fixture("evolve.json")["runs"])))
def test_oracle_evolve_matches_reference(idx):
    _check_run(I.fixture("evolve.json")["runs"][idx])


def test_oracle_assignments():
    fxs = I.fixture("assignments.json")
    for c in fxs["materialize"]:
        g, w = I.instance(c["inst"])
        orc = O.Oracle.of(g, w)
        grid, order = orc.materialize(np.array(c["groups"], dtype=np.int32))
        assert grid.tolist() == c["grid"] and list(order) == c["order"]
        o3, _ = orc.evaluate_assignment(grid)
        assert o3[0] == fx(c["total"]) and o3[1] == fx(c["datap"]) and o3[2] == fx(c["pipelinep"])
    for c in fxs["random"]:
        g, w = I.instance(c["inst"])
        rng = np.random.Generator(np.random.PCG64(0))
        s = rng.bit_generator.state
        s["state"]["state"], s["state"]["inc"] = int(c["state0"][0]), int(c["state0"][1])
        s["has_uint32"], s["uinteger"] = 0, 0
        rng.bit_generator.state = s
        st = O.PCG64State.from_generator(rng)
        grid = np.empty((w.d_dp, w.d_pp), dtype=np.int32)
        order = np.empty(w.d_pp, dtype=np.int32)
        import ctypes as C
        O.lib().orc_random_assignment(C.byref(st), g.n, w.d_pp, w.d_dp, grid, order)
        assert grid.tolist() == c["grid"] and list(order) == c["order"]
        o3, _ = O.Oracle.of(g, w).evaluate_assignment(grid)
        assert o3[0] == fx(c["total"])


@pytest.mark.parametrize("idx", range(len(I.fixture("evolve_1000.json")["runs"])))
def test_oracle_evolve_1000_generations(idx):
    """The GA time-to-converge anchors (pop 64, 1000 gens, ours, seed 0)."""
    _check_run(I.fixture("evolve_1000.json")["runs"][idx])


def test_oracle_config5_heuristic_and_passes():
    """Config 5 (1024 devices, 32 x 32): heuristic pricing and one pass of each
    flavour, as the reference computed them (tests/golden/big.json)."""
    from paper_2206_01288_b200.netmodel import random_graph
    from paper_2206_01288_b200.workload import WorkloadSpec
    g = random_graph(0, 1024)
    w = WorkloadSpec(32, 32, 268_435_456, 201_326_592)
    orc = O.Oracle.of(g, w)
    big = I.fixture("big.json")
    for c in big["heuristic_costs"]:
        t, d, p, order = orc.comm_cost_heuristic(np.array(c["groups"], dtype=np.int32))
        assert t == fx(c["total"]) and d == fx(c["datap"]) and p == fx(c["pipelinep"])
        assert list(order) == c["order"]
    for c in big["passes"]:
        st = O.rng_state(c["seed"])
        ch, out = orc.one_pass(np.array(c["groups"], dtype=np.int32), c["kind"], st, c["phase"])
        assert ch == c["changed"] and out.tolist() == c["out"]
        assert _rng_after(st) == c["rng_after"]


def test_oracle_matches_reference_config45_extra():
    """tests/golden/big_extra.npz: 32 config-4 and 12 config-5 layouts priced
    by the reference's comm_cost (make_golden_big.py)."""
    import numpy as np
    d = np.load(I.GOLDEN / "big_extra.npz")
    for name in ("config4", "config5"):
        g, w = I.instance(name)
        parts = d[f"{name}/parts"][:6]  # the oracle's k = 16 Held-Karp is the slow part
        t, dp, pp = O.Oracle.of(g, w).comm_cost_batch(parts, threads=O.cpu_count())
        assert np.array_equal(t, d[f"{name}/total"][:6]) and np.array_equal(dp, d[f"{name}/datap"][:6])
        assert np.array_equal(pp, d[f"{name}/pipelinep"][:6])
