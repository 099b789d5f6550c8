"""GPU parity of the fitness evaluator (K0 tables + K1 eval) through the C-ABI.

Every comparison is bitwise (==) against the oracle or against the golden
vectors the reference produced; no tolerance is applied anywhere.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from tests import _instances as I

pytestmark = pytest.mark.gpu

hs = pytest.importorskip("paper_2206_01288_b200")


def _gpu_names():
    return [n for n, m in I.meta().items() if m["recipe"]["w"][0] <= 16 and m["recipe"]["w"][1] <= 64]


@pytest.mark.parametrize("name", sorted(_gpu_names()))
def test_pair_tables_bitwise(name):
    from paper_2206_01288_b200 import _native as N
    g, w = I.instance(name)
    dp, pp, sw = N.instance_for(g, w).tables()
    odp, opp, osw = O.Oracle.of(g, w).tables()
    assert np.array_equal(dp, odp) and np.array_equal(pp, opp) and np.array_equal(sw, osw)


@pytest.mark.parametrize("name", sorted(_gpu_names()))
def test_batch_matches_reference_golden(name):
    g, w = I.instance(name)
    C = I.costs()
    parts = C[f"{name}/parts"]
    r = hs.comm_cost_batch(g, parts, w, per_group=True, order=True)
    assert np.array_equal(r["total"], C[f"{name}/total"])
    assert np.array_equal(r["datap"], C[f"{name}/datap"])
    assert np.array_equal(r["pipelinep"], C[f"{name}/pipelinep"])
    assert np.array_equal(r["per_group"], C[f"{name}/per_group"])
    assert np.array_equal(r["order"].astype(np.int16), C[f"{name}/order"])


def test_single_comm_cost_breakdown():
    g, w = I.instance("case5")
    C = I.costs()
    for i in range(5):
        p = hs.Partition.from_groups(C["case5/parts"][i].tolist())
        cb = hs.comm_cost(g, p, w)
        assert cb.total == C["case5/total"][i]
        assert cb.total == cb.datap + cb.pipelinep
        assert cb.per_group_datap == tuple(C["case5/per_group"][i])
        assert cb.pipeline_order.order == tuple(int(x) for x in C["case5/order"][i])
        assert cb.pipeline_order.total == cb.pipelinep


def test_g4_golden_values():
    g, w = I.instance("g4")
    good = hs.comm_cost(g, hs.Partition(((0, 1), (2, 3))), w)
    assert good.datap == 0.402 and good.pipelinep == 2.1
    assert good.total == pytest.approx(2.502, rel=1e-9)
    for p in (((0, 2), (1, 3)), ((0, 3), (1, 2))):
        bad = hs.comm_cost(g, hs.Partition(p), w)
        assert bad.datap == 4.1 and bad.pipelinep == 0.202


def _random_parts(seed, count, n, k, m):
    rng = np.random.default_rng(seed)
    return np.sort(rng.permuted(np.tile(np.arange(n, dtype=np.int16), (count, 1)), axis=1).reshape(count, k, m),
                   axis=2)


@pytest.mark.parametrize("case", [1, 2, 3, 4, 5])
def test_20k_layouts_per_case_bitwise_vs_oracle(case):
    g, w = I.instance(f"case{case}")
    parts = _random_parts(case, 20000, 64, 8, 8)
    r = hs.comm_cost_batch(g, parts, w)
    t, d, p = O.Oracle.of(g, w).comm_cost_batch(parts, threads=O.cpu_count())
    assert np.array_equal(r["total"], t)
    assert np.array_equal(r["datap"], d)
    assert np.array_equal(r["pipelinep"], p)


@pytest.mark.parametrize("case", [2, 4, 5])
def test_large_device_batch_with_malformed_rows_vs_oracle(case):
    """P = 50,003 in one device launch (a partial last quad), per-group
    values, and malformed rows scattered through it (NaN + count)."""
    import torch
    from paper_2206_01288_b200 import _native as N
    g, w = I.instance(f"case{case}")
    P = 50003
    parts = _random_parts(100 + case, P, 64, 8, 8)
    bad = [5, 31337, P - 1]
    parts[5, 0, 1] = parts[5, 0, 0]              # duplicate device
    parts[31337, 2, :] = parts[31337, 2, ::-1]  # not ascending
    parts[P - 1, 3, 7] = 64                      # out of range
    inst = N.instance_for(g, w)
    t = torch.from_numpy(parts).cuda()
    o = [torch.empty(P, dtype=torch.float64, device="cuda") for _ in range(3)]
    pg = torch.empty((P, 8), dtype=torch.float64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    N.check(N.lib().hs_eval_batch(inst.handle, t.data_ptr(), P, o[0].data_ptr(), o[1].data_ptr(), o[2].data_ptr(),
                                  pg.data_ptr(), None, cnt.data_ptr(), N.stream_ptr(inst.device)), "hs_eval_batch")
    tot, dp_, pp_, pg = (x.cpu().numpy() for x in (*o, pg))
    assert int(cnt.item()) == 3
    keep = np.setdiff1d(np.arange(P), bad)
    orc = O.Oracle.of(g, w)
    want_t, want_d, want_p = orc.comm_cost_batch(parts[keep], threads=O.cpu_count())
    assert np.array_equal(tot[keep], want_t)
    assert np.array_equal(dp_[keep], want_d)
    assert np.array_equal(pp_[keep], want_p)
    assert np.isnan(tot[bad]).all() and np.isnan(dp_[bad]).all() and np.isnan(pp_[bad]).all()
    for i in keep[::997]:
        assert np.array_equal(pg[i], orc.comm_cost(parts[i])[3])


@pytest.mark.parametrize("name", ["r64_8x8", "r36_6x6", "r64_2x32", "r48_3x16", "r40_4x10", "config1"])
def test_random_graphs_bitwise_vs_oracle(name):
    g, w = I.instance(name)
    parts = _random_parts(7, 3000, g.n, w.d_pp, w.d_dp)
    r = hs.comm_cost_batch(g, parts, w)
    t, d, p = O.Oracle.of(g, w).comm_cost_batch(parts, threads=O.cpu_count())
    assert np.array_equal(r["total"], t) and np.array_equal(r["datap"], d) and np.array_equal(r["pipelinep"], p)


def test_device_tensor_path_matches_host_path():
    import torch
    g, w = I.instance("case4")
    parts = _random_parts(11, 4096, 64, 8, 8)
    host = hs.comm_cost_batch(g, parts, w, per_group=True, order=True)
    dev = hs.comm_cost_batch(g, torch.from_numpy(parts).cuda(), w, per_group=True, order=True)
    for key in host:
        assert np.array_equal(host[key], dev[key].cpu().numpy()), key


def test_relabeling_groups_is_invariant_at_scale():
    g, w = I.instance("case5")
    parts = _random_parts(3, 8192, 64, 8, 8)
    rng = np.random.default_rng(0)
    shuffled = np.stack([p[rng.permutation(8)] for p in parts])
    a = hs.comm_cost_batch(g, parts, w)
    b = hs.comm_cost_batch(g, shuffled, w)
    for key in a:
        assert np.array_equal(a[key], b[key])


def test_chunked_host_path_crosses_chunk_boundary():
    g, w = I.instance("case2")
    parts = _random_parts(5, (1 << 18) + 1000, 64, 8, 8)
    r = hs.comm_cost_batch(g, parts, w)
    # host chunks (hs_eval_batch_host): per-launch 2^13 then 2^16, streamed 2^12 then 2^15
    b0, b1 = 1 << 13, (1 << 13) + (1 << 16)
    sel = np.r_[0:50, b0 - 25:b0 + 25, b1 - 25:b1 + 25, (1 << 18) - 25:(1 << 18) + 25, len(parts) - 50:len(parts)]
    t, _, _ = O.Oracle.of(g, w).comm_cost_batch(parts[sel], threads=O.cpu_count())
    assert np.array_equal(r["total"][sel], t)
    assert np.all(np.isfinite(r["total"]))


@pytest.mark.parametrize("case", [1, 2, 3, 4, 5])
def test_stage_order_and_per_group_at_8x8_vs_oracle(case):
    """comm_cost's full CostBreakdown at N = 64, 8x8 (per-group values and
    the stage order) == the oracle's, ties included (cases 1-3 have two
    distinct link costs)."""
    g, w = I.instance(f"case{case}")
    parts = _random_parts(900 + case, 3000, 64, 8, 8)
    r = hs.comm_cost_batch(g, parts, w, per_group=True, order=True)
    orc = O.Oracle.of(g, w)
    for i in range(0, len(parts), 7):
        tot, dp, pp, pg, order = orc.comm_cost(parts[i])
        assert r["total"][i] == tot and r["datap"][i] == dp and r["pipelinep"][i] == pp
        assert np.array_equal(r["per_group"][i], pg)
        assert r["order"][i].tolist() == order.tolist(), (i, r["order"][i], order)


@pytest.mark.parametrize("P", [1, 3, 4097, 36864, 100003])
def test_streamed_host_path_equals_device_path(P):
    """The host-buffer path at N = 64, 8x8 runs one kernel that consumes its
    chunks as they land (stream value writes / waits): odd sizes, sizes
    below one chunk, per-group outputs -- identical to the device path."""
    import torch
    g, w = I.instance("case4")
    parts = _random_parts(40 + P % 7, P, 64, 8, 8)
    host = hs.comm_cost_batch(g, parts, w, per_group=True)
    dev = hs.comm_cost_batch(g, torch.from_numpy(parts).cuda(), w, per_group=True)
    for key in host:
        assert np.array_equal(host[key], dev[key].cpu().numpy()), key


@pytest.mark.parametrize("P", [5, 70001])
def test_per_chunk_launch_host_path_equals_streamed(P, monkeypatch):
    """HS_HOST_STREAMED=0 (one eval8 launch per host chunk on alternating
    compute streams, read per call) prices exactly like the default streamed
    kernel, per-group outputs and a malformed row included."""
    g, w = I.instance("case5")
    parts = _random_parts(70 + P % 5, P, 64, 8, 8)
    a = hs.comm_cost_batch(g, parts, w, per_group=True)
    monkeypatch.setenv("HS_HOST_STREAMED", "0")
    b = hs.comm_cost_batch(g, parts, w, per_group=True)
    for key in a:
        assert np.array_equal(a[key], b[key]), key
    bad = parts.copy()
    bad[P // 2, 0, 0] = bad[P // 2, 1, 0]
    with pytest.raises(hs.CostModelError, match=f"1 of {P}"):
        hs.comm_cost_batch(g, bad, w)


def test_host_path_spans_more_than_its_device_buffers():
    """The host-buffer path holds up to 2^22 layouts on the device and runs
    larger batches span by span: 2^22 + 4,321 tiled layouts price exactly
    like their 997 distinct rows (oracle), in order, across the span seam."""
    g, w = I.instance("case3")
    uniq = _random_parts(31, 997, 64, 8, 8)
    P = (1 << 22) + 4321
    reps = -(-P // len(uniq))
    parts = np.tile(uniq, (reps, 1, 1))[:P]
    r = hs.comm_cost_batch(g, parts, w)
    t, _, _ = O.Oracle.of(g, w).comm_cost_batch(uniq, threads=O.cpu_count())
    want = np.tile(t, reps)[:P]
    assert np.array_equal(r["total"], want)


def test_malformed_partitions_raise():
    g, w = I.instance("case1")
    parts = _random_parts(1, 64, 64, 8, 8)
    bad = parts.copy()
    bad[3, 0, 0] = bad[3, 1, 0]  # duplicate device
    with pytest.raises(hs.CostModelError, match="1 of 64"):
        hs.comm_cost_batch(g, bad, w)
    bad = parts.copy()
    bad[5, 2] = bad[5, 2][::-1]  # descending members
    with pytest.raises(hs.CostModelError):
        hs.comm_cost_batch(g, bad, w)
    bad = parts.copy()
    bad[7, 0, 0] = 64  # out of range
    with pytest.raises(hs.CostModelError):
        hs.comm_cost_batch(g, bad, w)


def test_empty_batch():
    g, w = I.instance("case1")
    r = hs.comm_cost_batch(g, np.empty((0, 8, 8), dtype=np.int16), w)
    assert r["total"].shape == (0,)


def test_bottleneck_and_path_solvers_vs_golden():
    fxs = I.fixture("solvers.json")
    for c in fxs["matching"]:
        m = c["m"]
        wm = np.array([I.fx(x) for x in c["w"]]).reshape(m, m)
        assert hs.bottleneck_value(wm) == I.fx(c["value"])
    for c in fxs["tsp"]:
        k = c["k"]
        wm = np.array([I.fx(x) for x in c["w"]]).reshape(k, k)
        r = hs.open_loop_tsp(wm)
        assert r.total == I.fx(c["total"]) and list(r.order) == c["order"]


def test_batched_bottleneck_vs_oracle_with_ties():
    rng = np.random.default_rng(9)
    for m in (1, 2, 3, 5, 8, 13, 32, 64):
        stack = rng.integers(0, 6, size=(300, m, m)).astype(float) * 0.25
        got = hs.bottleneck_values(stack)
        want = np.array([O.bottleneck_value(x) for x in stack])
        assert np.array_equal(got, want), m


@pytest.mark.parametrize("name,count", [("r32_16x2", 300), ("r48_12x4", 200), ("r128_16x8", 100), ("config4", 12),
                                        ("r18_9x2", 300)])
def test_cta_path_d_pp_above_8_vs_oracle(name, count):
    """d_pp 9..16 (one CTA per candidate, global Held-Karp scratch) vs the oracle."""
    g, w = I.instance(name)
    parts = _random_parts(31, count, g.n, w.d_pp, w.d_dp)
    r = hs.comm_cost_batch(g, parts, w, per_group=True, order=True)
    orc = O.Oracle.of(g, w)
    t, d, p = orc.comm_cost_batch(parts, threads=O.cpu_count())
    assert np.array_equal(r["total"], t) and np.array_equal(r["datap"], d) and np.array_equal(r["pipelinep"], p)
    for i in range(min(count, 6)):
        tt, dd, pp, pg, order = orc.comm_cost(parts[i])
        assert np.array_equal(r["per_group"][i], pg) and list(r["order"][i]) == list(order)


def test_path_solver_k_9_to_16_vs_oracle():
    rng = np.random.default_rng(5)
    for k in (9, 12, 14, 16):
        stack = rng.uniform(0, 10, size=(6, k, k))
        stack = (stack + stack.transpose(0, 2, 1)) / 2.0
        for x in stack:
            np.fill_diagonal(x, 0.0)
        tot, order = hs.open_loop_tsps(stack)
        for i in range(len(stack)):
            o, t = O.open_loop_tsp(stack[i])
            assert tot[i] == t and tuple(order[i]) == o


@pytest.mark.parametrize("name", sorted(_gpu_names()))
def test_no_order_evaluator_matches_golden(name):
    """order=False prices with the two-layer Held-Karp schedule (no compact
    table kept, more warps per SM); same bits as the golden vectors."""
    g, w = I.instance(name)
    C = I.costs()
    parts = C[f"{name}/parts"]
    r = hs.comm_cost_batch(g, parts, w, per_group=True)
    assert np.array_equal(r["total"], C[f"{name}/total"])
    assert np.array_equal(r["datap"], C[f"{name}/datap"])
    assert np.array_equal(r["pipelinep"], C[f"{name}/pipelinep"])
    assert np.array_equal(r["per_group"], C[f"{name}/per_group"])


def test_no_order_evaluator_invalid_ragged_and_offset_views():
    import torch
    g, w = I.instance("case5")
    parts = _random_parts(21, 1000, 64, 8, 8)
    ref = O.Oracle.of(g, w).comm_cost_batch(parts, threads=O.cpu_count())[0]
    dev = torch.from_numpy(parts).cuda()
    assert np.array_equal(hs.comm_cost_batch(g, dev, w)["total"].cpu().numpy(), ref)
    assert np.array_equal(hs.comm_cost_batch(g, dev, w, order=True)["total"].cpu().numpy(), ref)
    # a view at a 2-byte offset
    buf = torch.empty(1000 * 64 + 1, dtype=torch.int16, device="cuda")
    buf[1:] = dev.reshape(-1)
    view = buf[1:].view(1000, 8, 8)
    assert np.array_equal(hs.comm_cost_batch(g, view, w)["total"].cpu().numpy(), ref)
    # malformed candidates scattered through the batch
    bad = parts.copy()
    for i in (0, 31, 32, 500, 999):
        bad[i, 3, 2] = bad[i, 3, 1]
    with pytest.raises(hs.CostModelError, match="5 of 1000"):
        hs.comm_cost_batch(g, bad, w)
    from paper_2206_01288_b200 import _native as N
    inst = N.instance_for(g, w)
    t = torch.from_numpy(bad).cuda()
    tot = torch.empty(1000, dtype=torch.float64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    N.check(N.lib().hs_eval_batch(inst.handle, t.data_ptr(), 1000, tot.data_ptr(), None, None, None, None,
                                  cnt.data_ptr(), N.stream_ptr(inst.device)), "hs_eval_batch")
    got = tot.cpu().numpy()
    assert int(cnt.item()) == 5
    good = np.ones(1000, bool)
    good[[0, 31, 32, 500, 999]] = False
    assert np.isnan(got[~good]).all()
    assert np.array_equal(got[good], ref[good])


@pytest.mark.parametrize("name,count", [("r32_16x2", 300), ("r48_12x4", 200), ("r128_16x8", 100), ("config4", 40),
                                        ("r18_9x2", 300)])
def test_cluster_held_karp_no_order_vs_oracle(name, count):
    """order=False at d_pp 9..16: stage kernel + cluster Held-Karp (two live
    layers in distributed shared memory) vs the oracle, bit for bit."""
    g, w = I.instance(name)
    parts = _random_parts(37, count, g.n, w.d_pp, w.d_dp)
    r = hs.comm_cost_batch(g, parts, w, per_group=True)
    t, d, p = O.Oracle.of(g, w).comm_cost_batch(parts, threads=O.cpu_count())
    assert np.array_equal(r["total"], t) and np.array_equal(r["datap"], d) and np.array_equal(r["pipelinep"], p)
    full = hs.comm_cost_batch(g, parts[:8], w, per_group=True, order=True)
    assert np.array_equal(r["per_group"][:8], full["per_group"])


@pytest.mark.parametrize("k", [9, 12, 13, 14, 15, 16])
def test_cluster_held_karp_every_cluster_size(k):
    """k = 9..13 fit one CTA, 14 / 15 / 16 split the live layers over 2 / 4 / 8."""
    from paper_2206_01288_b200.netmodel import random_graph
    from paper_2206_01288_b200.workload import WorkloadSpec
    g = random_graph(100 + k, 3 * k)
    w = WorkloadSpec(k, 3, 1 << 30, 3 << 26)
    parts = _random_parts(k, 64, g.n, k, 3)
    r = hs.comm_cost_batch(g, parts, w)
    t, d, p = O.Oracle.of(g, w).comm_cost_batch(parts, threads=O.cpu_count())
    assert np.array_equal(r["total"], t) and np.array_equal(r["pipelinep"], p)


def test_cluster_held_karp_device_batch_with_malformed_rows():
    """Device-tensor input: malformed rows are counted and raise, like the CTA path."""
    import torch
    g, w = I.instance("config4")
    parts = _random_parts(41, 20, g.n, w.d_pp, w.d_dp)
    bad = parts.copy()
    bad[3, 0, 0], bad[3, 0, 1] = bad[3, 0, 1], bad[3, 0, 0]  # not ascending
    with pytest.raises(hs.CostModelError):
        hs.comm_cost_batch(g, torch.from_numpy(bad).cuda(), w)
    r = hs.comm_cost_batch(g, torch.from_numpy(parts).cuda(), w)
    t, d, p = O.Oracle.of(g, w).comm_cost_batch(parts, threads=O.cpu_count())
    assert np.array_equal(r["total"].cpu().numpy(), t)


def _devices_for_split():
    import torch
    n = torch.cuda.device_count()
    return list(range(n)) if n > 1 else [0, 0]


@pytest.mark.parametrize("name", ["case5", "config4"])
def test_multi_device_split_is_bitwise_single_device(name):
    """comm_cost_batch(devices=[...]) shards contiguously over GPUs (or two
    host threads on one GPU) and must equal the single-device result."""
    g, w = I.instance(name)
    P = 20_001 if w.d_pp <= 8 else 301
    parts = _random_parts(21, P, g.lat.shape[0], w.d_pp, w.d_dp)
    one = hs.comm_cost_batch(g, parts, w, per_group=True)
    devs = _devices_for_split()
    many = hs.comm_cost_batch(g, parts, w, per_group=True, devices=devs)
    for key in one:
        assert np.array_equal(one[key], many[key]), key


def test_multi_device_split_device_tensor_and_errors():
    import torch
    g, w = I.instance("case3")
    parts = _random_parts(22, 5003, 64, 8, 8)
    ref = hs.comm_cost_batch(g, parts, w)["total"]
    got = hs.comm_cost_batch(g, torch.from_numpy(parts).cuda(), w, devices=_devices_for_split())["total"]
    assert got.device.type == "cuda" and np.array_equal(got.cpu().numpy(), ref)
    bad = parts.copy()
    bad[-1, 0, 0] = bad[-1, 0, 1]
    with pytest.raises(hs.CostModelError, match="1 of 5003"):
        hs.comm_cost_batch(g, bad, w, devices=_devices_for_split())


def test_two_streams_concurrently_on_one_config4_handle():
    """Per-handle re-entrancy: d_pp = 16 calls on two
    streams of one handle run concurrently with private scratch sets, the
    stage-kernel + cluster path (no order) on one and the CTA path (with
    order) on the other, twice each; all must equal the oracle."""
    import torch

    from paper_2206_01288_b200 import _native as N
    from paper_2206_01288_b200.costmodel import _launch_device
    g, w = I.instance("config4")
    inst = N.instance_for(g, w)
    a = _random_parts(31, 24, 512, 16, 32)
    b = _random_parts(32, 24, 512, 16, 32)
    orc = O.Oracle.of(g, w)
    want_a = orc.comm_cost_batch(a, threads=O.cpu_count())[0]
    want_b = orc.comm_cost_batch(b, threads=O.cpu_count())[0]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    torch.cuda.synchronize()
    outs = []
    for _ in range(2):
        with torch.cuda.stream(s1):
            outs.append(("a", _launch_device(inst, ta, False, False)))
        with torch.cuda.stream(s2):
            outs.append(("b", _launch_device(inst, tb, True, True)))
    torch.cuda.synchronize()
    for which, (out, bad) in outs:
        assert int(bad.item()) == 0
        want = want_a if which == "a" else want_b
        assert np.array_equal(out["total"].cpu().numpy(), want), which


def test_host_path_from_two_threads_on_one_handle():
    from concurrent.futures import ThreadPoolExecutor
    g, w = I.instance("case1")
    pops = [_random_parts(40 + i, 70_000, 64, 8, 8) for i in range(4)]
    ref = [hs.comm_cost_batch(g, p, w)["total"] for p in pops]
    with ThreadPoolExecutor(4) as ex:
        got = list(ex.map(lambda p: hs.comm_cost_batch(g, p, w)["total"], pops))
    for r, x in zip(ref, got):
        assert np.array_equal(r, x)


@pytest.mark.parametrize("name", ["config4", "config5"])
def test_config45_extra_reference_vectors(name):
    """Every reference-priced config-4/5 layout of big_extra.npz, through the
    stage + cluster path (no order) and the CTA path (order, per-group)."""
    d = np.load(I.GOLDEN / "big_extra.npz")
    g, w = I.instance(name)
    parts = d[f"{name}/parts"]
    fast = hs.comm_cost_batch(g, parts, w)
    full = hs.comm_cost_batch(g, parts, w, per_group=True, order=True)
    for r in (fast, full):
        assert np.array_equal(r["total"], d[f"{name}/total"])
        assert np.array_equal(r["datap"], d[f"{name}/datap"])
        assert np.array_equal(r["pipelinep"], d[f"{name}/pipelinep"])
    assert np.array_equal(full["per_group"], d[f"{name}/per_group"])
    assert np.array_equal(full["order"], d[f"{name}/order"])
