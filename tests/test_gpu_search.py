"""GPU parity of the search path (K2 gains / local search, K3 GA) through the C-ABI.

Bitwise against the golden vectors the reference produced and, at larger
scale, against the oracle; RNG states must come back advanced exactly as
numpy would advance them.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from tests import _instances as I
from tests._instances import fx

pytestmark = pytest.mark.gpu

hs = pytest.importorskip("paper_2206_01288_b200")
from paper_2206_01288_b200 import scheduler as S  # noqa: E402


def _rng_tuple(rng):
    st = rng.bit_generator.state
    return [str(st["state"]["state"]), st["has_uint32"], st["uinteger"]]


def _gpu_ok(name):
    k, m = I.meta()[name]["recipe"]["w"][:2]
    return k <= 16 and m <= 64


def test_surrogate_weights_and_g4_gains():
    g, w = I.instance("g4")
    sw = S.SurrogateWeights.from_instance(g, w)
    assert sw.w[0, 1] == pytest.approx(0.501, rel=1e-12) and sw.w[0, 2] == pytest.approx(5.05, rel=1e-12)
    good, bad = hs.Partition(((0, 1), (2, 3))), hs.Partition(((0, 2), (1, 3)))
    assert S.gain_ours(sw, bad, 0, 1, (0, 2, 1, 3)) == pytest.approx(-4.549, rel=1e-9)
    assert S.gain_ours(sw, good, 0, 1, (0, 1, 2, 3)) == pytest.approx(9.098, rel=1e-9)
    assert S.gain_kl(sw, good, 0, 2) == pytest.approx(9.098, rel=1e-9)
    with pytest.raises(S.ScheduleError, match="both in group 0"):
        S.gain_kl(sw, good, 0, 1)


def test_gains_match_golden():
    for c in I.fixture("search.json")["gains"]:
        g, w = I.instance(c["inst"])
        sw = S.SurrogateWeights.from_instance(g, w)
        p = hs.Partition.from_groups(c["groups"])
        if c["kind"] == "ours":
            j, j2, *cand = c["args"]
            v = S.gain_ours(sw, p, j, j2, tuple(cand))
        else:
            v = S.gain_kl(sw, p, *c["args"])
        assert v == fx(c["value"]), c


def test_gain_kl_equals_cut_difference_dyadic():
    rng = np.random.default_rng(0)
    for _ in range(50):
        raw = rng.integers(0, 256, size=(12, 12)).astype(float)
        wm = (raw + raw.T) / 16.0
        np.fill_diagonal(wm, 0.0)
        sw = S.SurrogateWeights(wm)
        perm = rng.permutation(12)
        p = hs.Partition.from_groups(perm.reshape(3, 4).tolist())
        ja, jb = rng.choice(3, size=2, replace=False)
        d = int(rng.choice(p.groups[ja]))
        d2 = int(rng.choice(p.groups[jb]))
        cut = lambda ga, gb: sum(wm[x, y] for x in ga for y in gb)
        before = cut(p.groups[ja], p.groups[jb])
        after = cut([x for x in p.groups[ja] if x != d] + [d2], [x for x in p.groups[jb] if x != d2] + [d])
        assert S.gain_kl(sw, p, d, d2) == before - after


def test_passes_match_golden():
    for c in I.fixture("search.json")["passes"]:
        if not _gpu_ok(c["inst"]):
            continue
        g, w = I.instance(c["inst"])
        rng = np.random.Generator(np.random.PCG64(c["seed"]))
        ch, out = S.refine_pass(g, w, hs.Partition.from_groups(c["groups"]), c["kind"], rng, c["phase"])
        assert ch == c["changed"], (c["inst"], c["kind"], c["phase"])
        assert [list(x) for x in out.groups] == [sorted(x) for x in c["out"]], (c["inst"], c["kind"], c["phase"])
        assert _rng_tuple(rng) == c["rng_after"]


def test_crossover_matches_golden():
    for c in I.fixture("search.json")["crossover"]:
        rng = np.random.Generator(np.random.PCG64(c["seed"]))
        child = S.crossover(hs.Partition.from_groups(c["p1"]), hs.Partition.from_groups(c["p2"]), rng)
        assert [list(x) for x in child.groups] == c["child"]
        assert _rng_tuple(rng) == c["rng_after"]


def test_crossover_identical_parents_is_copy_and_balanced():
    good = hs.Partition(((0, 1), (2, 3)))
    assert S.crossover(good, good, np.random.default_rng(0)) == good
    rng = np.random.default_rng(42)
    for _ in range(50):
        p1 = S.random_partition(rng, 12, 3, 4)
        p2 = S.random_partition(rng, 12, 3, 4)
        child = S.crossover(p1, p2, rng)
        assert sorted(d for grp in child.groups for d in grp) == list(range(12))


def test_local_search_matches_golden():
    for c in I.fixture("search.json")["local_search"]:
        if not _gpu_ok(c["inst"]):
            continue
        g, w = I.instance(c["inst"])
        rng = np.random.default_rng(c["seed"])
        out = S.local_search(g, w, hs.Partition.from_groups(c["groups"]), kind=c["kind"], rng=rng)
        assert [list(x) for x in out.groups] == c["out"], (c["inst"], c["kind"])
        assert _rng_tuple(rng) == c["rng_after"]


def test_init_population_matches_numpy_draws():
    g, w = I.instance("case5")
    cfg = S.ScheduleConfig(pop_size=16, seed=3)
    pop = S.init_population(g, w, cfg)
    rng = np.random.Generator(np.random.PCG64(3))
    for p in pop:
        perm = rng.permutation(64)
        assert [list(x) for x in p.groups] == [sorted(perm[j * 8:(j + 1) * 8].tolist()) for j in range(8)]


def _check_result(res, run):
    d = res.to_dict()
    assert d["partition"] == run["partition"]
    assert d["cost"]["total"] == fx(run["total"])
    assert d["cost"]["datap"] == fx(run["datap"]) and d["cost"]["pipelinep"] == fx(run["pipelinep"])
    assert d["cost"]["per_group_datap"] == [fx(x) for x in run["per_group"]]
    assert d["cost"]["pipeline_order"] == run["order"]
    assert d["evaluations"] == run["evaluations"]
    assert [r[1] for r in d["trace"]] == [fx(x) for x in run["trace_best"]]
    assert [r[2] for r in d["trace"]] == [fx(x) for x in run["trace_mean"]]


@pytest.mark.parametrize("idx", range(len(I.fixture("evolve.json")["runs"])))
def test_evolve_matches_reference_golden(idx):
    run = I.fixture("evolve.json")["runs"][idx]
    if not _gpu_ok(run["inst"]):
        pytest.skip("shape beyond the GPU GA")
    g, w = I.instance(run["inst"])
    cfg = S.ScheduleConfig(pop_size=run["pop"], generations=run["gens"], local_search=run["kind"], seed=run["seed"],
                           patience=run["patience"])
    _check_result(S.evolve(g, w, cfg), run)


@pytest.mark.parametrize("idx", range(len(I.fixture("evolve_1000.json")["runs"])))
def test_evolve_1000_generations_matches_reference(idx):
    """GA time-to-converge anchors: identical trace, partition, evaluations."""
    run = I.fixture("evolve_1000.json")["runs"][idx]
    g, w = I.instance(run["inst"])
    cfg = S.ScheduleConfig(pop_size=run["pop"], generations=run["gens"], local_search=run["kind"], seed=run["seed"])
    _check_result(S.evolve(g, w, cfg), run)


@pytest.mark.parametrize("case", [1, 3, 4, 5])
def test_islands_equal_independent_runs_vs_oracle(case):
    """48 islands in one launch == 48 oracle evolve runs with the same streams."""
    g, w = I.instance(f"case{case}")
    cfg = S.ScheduleConfig(pop_size=16, generations=30, local_search="ours" if case % 2 else "kl")
    rngs = S.island_seeds(case, 48)
    states = [O.PCG64State.from_generator(r) for r in S.island_seeds(case, 48)]
    sess = S.GASession(g, w, cfg, rngs)
    sess.run(cfg.generations)
    res = sess.results()
    orc = O.Oracle.of(g, w)
    for i, r in enumerate(res):
        o = orc.evolve(cfg.pop_size, cfg.generations, cfg.local_search, state=states[i])
        assert [list(x) for x in r.best_partition.groups] == o["partition"].tolist()
        assert r.best_cost.total == o["total"] and r.evaluations == o["evaluations"]
        assert [t[1] for t in r.trace] == list(o["trace_best"])
        assert [t[2] for t in r.trace] == list(o["trace_mean"])
        assert O.PCG64State.from_generator(rngs[i]).as_tuple() == states[i].as_tuple()


def test_epochs_equal_single_launch():
    g, w = I.instance("case5")
    cfg = S.ScheduleConfig(pop_size=32, generations=40, local_search="ours", seed=9)
    one = S.evolve(g, w, cfg)
    sess = S.GASession(g, w, cfg, [np.random.Generator(np.random.PCG64(9))])
    for until in (7, 19, 33, 40):
        sess.run(until)
    assert sess.results()[0].to_dict() == one.to_dict()


def test_migration_is_deterministic_and_keeps_best_monotone():
    g, w = I.instance("case5")
    cfg = S.ScheduleConfig(pop_size=16, generations=30, local_search="kl")

    def run():
        sess = S.GASession(g, w, cfg, S.island_seeds(1, 8))
        for epoch in range(3):
            sess.run(10 * (epoch + 1))
            gr, co = sess.export_elites(2)
            sess.import_elites(gr, co, [(i - 1) % 8 for i in range(8)])
        return sess.results()

    a, b = run(), run()
    assert [r.to_dict() for r in a] == [r.to_dict() for r in b]
    for r in a:
        best = [t[1] for t in r.trace]
        assert all(y <= x for x, y in zip(best, best[1:]))
        assert r.best_cost.total == hs.comm_cost(g, r.best_partition, w).total


def test_evolve_errors_like_reference():
    g, w = I.instance("r4_1x4")
    with pytest.raises(ValueError):
        S.evolve(g, w, S.ScheduleConfig(pop_size=4, generations=3, local_search="ours"))
    res = S.evolve(g, w, S.ScheduleConfig(pop_size=4, generations=3, local_search="kl"))
    assert res.best_cost.pipelinep == 0.0


@pytest.mark.parametrize("name,kind,pop,gens", [("r32_16x2", "ours", 8, 12), ("r32_16x2", "kl", 8, 12),
                                                ("r48_12x4", "ours", 8, 6), ("r18_9x2", "ours", 8, 15),
                                                ("config4", "kl", 4, 2), ("config4", "ours", 4, 3),
                                                ("r64_2x32", "ours", 8, 12)])
def test_evolve_d_pp_above_8_vs_oracle(name, kind, pop, gens):
    """GA with CTA-level pricing (d_pp 9..16) or 32-member groups (the
    incremental fast-edge path) reproduces the oracle's evolve."""
    g, w = I.instance(name)
    cfg = S.ScheduleConfig(pop_size=pop, generations=gens, local_search=kind, seed=4)
    r = S.evolve(g, w, cfg)
    o = O.Oracle.of(g, w).evolve(pop, gens, kind, seed=4)
    assert [list(x) for x in r.best_partition.groups] == o["partition"].tolist()
    assert r.best_cost.total == o["total"] and r.evaluations == o["evaluations"]
    assert list(r.best_cost.pipeline_order.order) == list(o["order"])
    assert [t[1] for t in r.trace] == list(o["trace_best"])
    assert [t[2] for t in r.trace] == list(o["trace_mean"])


@pytest.mark.parametrize("name,kind,patience", [("r32_16x2", "ours", None), ("r48_12x4", "kl", 3),
                                                 ("r18_9x2", "ours", 4)])
def test_batch_priced_islands_d_pp_above_8_vs_oracle(name, kind, patience):
    """d_pp 9..16 islands with batch-priced generations (every island's
    snapshots of a generation priced together by the stage + cluster
    Held-Karp kernels), run in epochs, == independent oracle evolve runs."""
    g, w = I.instance(name)
    cfg = S.ScheduleConfig(pop_size=8, generations=10, local_search=kind, patience=patience)
    rngs = S.island_seeds(11, 12)
    states = [O.PCG64State.from_generator(r) for r in S.island_seeds(11, 12)]
    sess = S.GASession(g, w, cfg, rngs)
    for until in (3, 4, 10):
        sess.run(until)
    res = sess.results()
    orc = O.Oracle.of(g, w)
    for i, r in enumerate(res):
        o = orc.evolve(cfg.pop_size, cfg.generations, kind, state=states[i], patience=patience)
        assert [list(x) for x in r.best_partition.groups] == o["partition"].tolist()
        assert r.best_cost.total == o["total"] and r.evaluations == o["evaluations"]
        assert [t[1] for t in r.trace] == list(o["trace_best"])
        assert [t[2] for t in r.trace] == list(o["trace_mean"])
        assert O.PCG64State.from_generator(rngs[i]).as_tuple() == states[i].as_tuple()


def test_batch_priced_generations_equal_in_kernel_pricing(monkeypatch):
    """HS_GA_BATCH=0 (each island prices its snapshots in-kernel, one at a
    time) and the batch-priced generations give identical sessions,
    migration included."""
    g, w = I.instance("r32_16x2")
    cfg = S.ScheduleConfig(pop_size=8, generations=6, local_search="ours")

    def run():
        sess = S.GASession(g, w, cfg, S.island_seeds(2, 6))
        for epoch in range(2):
            sess.run(3 * (epoch + 1))
            gr, co = sess.export_elites(2)
            sess.import_elites(gr, co, [(i - 1) % 6 for i in range(6)])
        return [r.to_dict() for r in sess.results()]

    batched = run()
    monkeypatch.setenv("HS_GA_BATCH", "0")
    assert run() == batched


def test_local_search_d_pp_16_vs_oracle():
    g, w = I.instance("r32_16x2")
    rng = np.random.default_rng(1)
    for t in range(3):
        p = S.random_partition(rng, g.n, w.d_pp, w.d_dp)
        for kind in ("ours", "kl"):
            r1 = np.random.default_rng(50 + t)
            st = O.rng_state(np.random.default_rng(50 + t))
            out = S.local_search(g, w, p, kind=kind, rng=r1)
            want = O.Oracle.of(g, w).local_search(np.array(p.groups, dtype=np.int32), kind, st)
            assert [list(x) for x in out.groups] == want.tolist()


@pytest.mark.parametrize("kind", ["ours", "kl"])
def test_batch_priced_local_search_d_pp_16(kind, monkeypatch):
    """hs_local_search on 12 config-4 partitions: the passes' snapshots of
    all partitions priced in one batch (stage + cluster Held-Karp) == the
    in-kernel pricing (HS_GA_BATCH=0) == the oracle's local_search."""
    from paper_2206_01288_b200 import _native as N
    g, w = I.instance("config4")
    rng = np.random.default_rng(8)
    parts = np.stack([np.array(S.random_partition(rng, g.n, w.d_pp, w.d_dp).groups, dtype=np.int16)
                      for _ in range(12)])
    inst = N.instance_for(g, w)

    def run():
        st = S._states([np.random.default_rng(300 + i) for i in range(len(parts))])
        out = np.empty_like(parts)
        tot = np.empty(len(parts))
        ev = np.empty(len(parts), dtype=np.int32)
        N.check(N.lib().hs_local_search(inst.handle, S._KIND[kind], 8, len(parts), parts.ctypes.data, st,
                                        out.ctypes.data, tot.ctypes.data, ev.ctypes.data), "hs_local_search")
        return out, tot, ev

    batched = run()
    monkeypatch.setenv("HS_GA_BATCH", "0")
    in_kernel = run()
    for x, y in zip(batched, in_kernel):
        assert np.array_equal(x, y)
    orc = O.Oracle.of(g, w)
    for i in range(3):
        want = orc.local_search(parts[i].astype(np.int32), kind, O.rng_state(np.random.default_rng(300 + i)))
        assert batched[0][i].tolist() == want.tolist()


@pytest.mark.parametrize("kind", ["ours", "kl", "none"])
def test_warp_island_mode_equals_cta_mode(kind):
    """One warp per island gives the same results as one CTA per island."""
    g, w = I.instance("case5")
    cfg = S.ScheduleConfig(pop_size=16, generations=20, local_search=kind)
    a = S.GASession(g, w, cfg, S.island_seeds(3, 37), mode="cta")
    b = S.GASession(g, w, cfg, S.island_seeds(3, 37), mode="warp")
    a.run(cfg.generations)
    b.run(cfg.generations)
    ra, rb = a.results(), b.results()
    assert [r.to_dict() for r in ra] == [r.to_dict() for r in rb]


# Shapes around the register-resident driver paths: the d_dp = 8 sweep
# (n <= 128) and the chain rounds (n <= 64, k <= 8; 9- or 16-member unrolls),
# plus shapes that fall back to the shared-memory driver on either side.
DRIVER_SHAPES = [(32, 4, 8), (48, 6, 8), (48, 4, 12), (60, 5, 12), (45, 3, 15), (64, 4, 16), (64, 2, 32),
                 (96, 12, 8), (128, 16, 8), (40, 8, 5), (24, 8, 3)]


def _two_level(n, k):
    # few distinct weights (tie-heavy, like the preset data-centre cases)
    from paper_2206_01288_b200.netmodel import scenario_from_ms_gbps
    size = n // k
    return scenario_from_ms_gbps([(size, 0.1, 100.0)] * k, 0.25, 25.0, 0).graph()


@pytest.mark.parametrize("n,k,m", DRIVER_SHAPES)
@pytest.mark.parametrize("ties", [False, True])
def test_evolve_driver_shapes_vs_oracle(n, k, m, ties):
    """evolve (ours) through the register driver paths reproduces the oracle."""
    from paper_2206_01288_b200.netmodel import random_graph
    from paper_2206_01288_b200.workload import WorkloadSpec
    g = _two_level(n, k) if ties else random_graph(11 + n + k, n)
    w = WorkloadSpec(k, m, 1 << 30, 3 << 26)
    pop, gens = (8, 6) if k > 8 else (12, 25)
    cfg = S.ScheduleConfig(pop_size=pop, generations=gens, local_search="ours", seed=5)
    r = S.evolve(g, w, cfg)
    o = O.Oracle.of(g, w).evolve(pop, gens, "ours", seed=5)
    assert [list(x) for x in r.best_partition.groups] == o["partition"].tolist()
    assert r.best_cost.total == o["total"] and r.evaluations == o["evaluations"]
    assert [t[1] for t in r.trace] == list(o["trace_best"])
    assert [t[2] for t in r.trace] == list(o["trace_mean"])


@pytest.mark.parametrize("n,k,m", [(32, 4, 8), (48, 4, 12), (64, 8, 8), (128, 16, 8)])
def test_local_search_driver_shapes_vs_oracle(n, k, m):
    """local_search (ours) from random starts, RNG stream included."""
    from paper_2206_01288_b200.netmodel import random_graph
    from paper_2206_01288_b200.workload import WorkloadSpec
    g = random_graph(3 * n + k, n)
    w = WorkloadSpec(k, m, 1 << 30, 3 << 26)
    rng = np.random.default_rng(n)
    for t in range(4):
        p = S.random_partition(rng, n, k, m)
        r1 = np.random.default_rng(90 + t)
        st = O.rng_state(np.random.default_rng(90 + t))
        out = S.local_search(g, w, p, kind="ours", rng=r1)
        want = O.Oracle.of(g, w).local_search(np.array(p.groups, dtype=np.int32), "ours", st)
        assert [list(x) for x in out.groups] == want.tolist()


@pytest.mark.parametrize("case", [2, 4, 5])
@pytest.mark.parametrize("seed", [11, 12, 13, 14])
def test_evolve_paper_shape_seeds_vs_oracle(case, seed):
    """The paper shape (64 devices, 8x8) over several seeds: every chain-round
    shortcut (single-move rejection, lock-only rounds, prefix replay) and the
    sweep waves against the oracle's evolve, traces included."""
    g, w = I.instance(f"case{case}")
    cfg = S.ScheduleConfig(pop_size=16, generations=40, local_search="ours", seed=seed)
    r = S.evolve(g, w, cfg)
    o = O.Oracle.of(g, w).evolve(16, 40, "ours", seed=seed)
    assert [list(x) for x in r.best_partition.groups] == o["partition"].tolist()
    assert r.best_cost.total == o["total"] and r.evaluations == o["evaluations"]
    assert [t[1] for t in r.trace] == list(o["trace_best"])
    assert [t[2] for t in r.trace] == list(o["trace_mean"])


def test_ga_session_results_sync_and_partial_run_errors():
    """hs_ga_result drains the session's own (non-blocking) stream before it
    reads island states, and refuses a session that is not run to the end."""
    import torch

    from paper_2206_01288_b200 import _native as N
    g, w = I.instance("case5")
    cfg = S.ScheduleConfig(pop_size=32, generations=40, local_search="ours", seed=9)
    one = S.evolve(g, w, cfg)
    side = torch.cuda.Stream()
    sess = S.GASession(g, w, cfg, [np.random.Generator(np.random.PCG64(9))])
    sess.run(20, stream=side.cuda_stream)
    with pytest.raises(N.NativeError, match="not finished"):
        sess.results()
    sess.run(40, stream=side.cuda_stream)  # no host synchronisation before results()
    assert sess.results()[0].to_dict() == one.to_dict()


@pytest.mark.parametrize("name,kind,pop,gens,patience,max_passes",
                         [("case5", "ours", 16, 120, None, 8), ("case2", "ours", 64, 80, None, 8),
                          ("case4", "ours", 32, 150, 6, 8), ("case3", "kl", 24, 90, None, 8),
                          ("case1", "none", 16, 70, 9, 8), ("r24_3x8", "ours", 12, 60, None, 5),
                          ("r16_4x4", "ours", 20, 60, 4, 3), ("config1", "ours", 64, 100, None, 8)])
def test_speculative_pipeline_equals_oracle(name, kind, pop, gens, patience, max_passes):
    """One evolve runs as the speculative cluster pipeline (hs_search_ga_spec.cu):
    stream-position mispredictions (case 2: two sweep passes, predicted
    four), parent replacements under in-flight jobs, patience stops and
    epoch boundaries must leave the trace, result, evaluations and the
    caller's stream exactly those of the oracle."""
    g, w = I.instance(name)
    cfg = S.ScheduleConfig(pop_size=pop, generations=gens, local_search=kind, seed=11, patience=patience,
                           max_passes=max_passes)
    o = O.Oracle.of(g, w).evolve(pop, gens, kind, seed=11, max_passes=max_passes, patience=patience)
    r = S.evolve(g, w, cfg)
    assert [list(x) for x in r.best_partition.groups] == o["partition"].tolist()
    assert r.best_cost.total == o["total"] and r.evaluations == o["evaluations"]
    assert [t[1] for t in r.trace] == list(o["trace_best"])
    assert [t[2] for t in r.trace] == list(o["trace_mean"])
    # the same run in epochs (several launches of the pipeline)
    rng = np.random.Generator(np.random.PCG64(11))
    sess = S.GASession(g, w, cfg, [rng])
    for until in (gens // 3, gens // 2, gens):
        sess.run(until)
    assert sess.results()[0].to_dict() == r.to_dict()
