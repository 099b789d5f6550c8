"""Bi-level communication cost of balanced partitions, evaluated on the GPU.

Drop-in mirror of hetsched/costmodel.py's hot-path surface:
``Partition`` (:47-95), ``CostBreakdown`` (:114-131), ``comm_cost``
(:217-229), ``datap_cost`` (:171-175), ``pipeline_cost`` (:211-214), plus the
batch entry point ``comm_cost_batch`` that the GPU path adds.  Every cost
is computed by the sm_100a kernels in lib/libhetsched_sm100a.so (K0 pair
tables + K1 warp-per-candidate evaluator); Python only validates, packs
int16 layouts and unpacks results.  Results are bit-identical to the
reference (tests/test_gpu_costmodel.py).

Graphs and workloads are duck-typed: anything with ``lat``/``bw`` arrays and
``d_pp``/``d_dp``/``c_pp``/``c_dp`` works, including the reference's own
dataclasses.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable

import numpy as np

from . import _native as N
from .combinatorics import MatchingResult, PathResult, bottleneck_matchings, open_loop_tsp
from .workload import validate_workload


class CostModelError(ValueError):
    """Partition inconsistent with the network or the workload."""


@dataclass(frozen=True)
class Partition:
    """Balanced partition of devices 0..N-1; members ascending, group order kept."""

    groups: tuple[tuple[int, ...], ...]

    def __post_init__(self) -> None:
        groups = tuple(tuple(sorted(int(d) for d in grp)) for grp in self.groups)
        if not groups or not groups[0]:
            raise CostModelError("partition needs at least one non-empty group")
        if len({len(g) for g in groups}) != 1:
            raise CostModelError(f"unbalanced groups: sizes {sorted(len(g) for g in groups)}")
        flat = sorted(d for g in groups for d in g)
        if flat != list(range(len(flat))):
            raise CostModelError("groups must be disjoint and cover devices 0..N-1 exactly")
        object.__setattr__(self, "groups", groups)

    @property
    def d_pp(self) -> int:
        return len(self.groups)

    @property
    def d_dp(self) -> int:
        return len(self.groups[0])

    @property
    def n(self) -> int:
        return self.d_pp * self.d_dp

    def canonical(self) -> "Partition":
        return Partition(tuple(sorted(self.groups)))

    def key(self) -> tuple[tuple[int, ...], ...]:
        return tuple(sorted(self.groups))

    @classmethod
    def from_groups(cls, groups: Iterable[Iterable[int]]) -> "Partition":
        return cls(tuple(tuple(g) for g in groups))

    def as_array(self) -> np.ndarray:
        return np.asarray(self.groups, dtype=np.int16)


@dataclass(frozen=True)
class CostBreakdown:
    datap: float
    pipelinep: float
    total: float
    per_group_datap: tuple[float, ...]
    pipeline_order: PathResult

    def to_dict(self) -> dict:
        return {
            "datap": self.datap,
            "pipelinep": self.pipelinep,
            "total": self.total,
            "per_group_datap": list(self.per_group_datap),
            "pipeline_order": list(self.pipeline_order.order),
        }


@dataclass(frozen=True)
class CoarsenedGraph:
    """One vertex per group; edge_cost[j, j2] is the bottleneck of the pair
    matrix rows sorted(group j) x columns sorted(group j2), matchings[(j, j2)]
    (j < j2) its lexicographically smallest optimal pairing
    (costmodel.py:99-111)."""

    edge_cost: np.ndarray
    matchings: dict

    @property
    def k(self) -> int:
        return self.edge_cost.shape[0]


def _check_partition(p, g, w) -> None:
    n = len(p.groups) * len(p.groups[0])
    if n != g.lat.shape[0]:
        raise CostModelError(f"partition covers {n} devices but the network has {g.lat.shape[0]}")
    if len(p.groups) != w.d_pp or len(p.groups[0]) != w.d_dp:
        raise CostModelError(
            f"partition shape {len(p.groups)}x{len(p.groups[0])} does not match workload {w.d_pp}x{w.d_dp}")


def shard_bounds(P: int, G: int) -> list[tuple[int, int]]:
    """Contiguous split of P candidates over G devices:
    the first P % G shards hold one extra candidate; empty shards are kept
    so shard i always belongs to device i."""
    if G < 1:
        raise ValueError("need at least one device")
    base, extra = divmod(int(P), G)
    out, lo = [], 0
    for i in range(G):
        hi = lo + base + (1 if i < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def comm_cost_batch(g, groups, w, *, per_group: bool = False, order: bool = False, device: int | None = None,
                    heuristic: bool = False, devices=None):
    """Costs of a batch of partitions in one GPU pass.

    ``groups``: int16-compatible [P, d_pp, d_dp] with ascending members --
    a numpy array (host path: pinned staging, chunked H2D / kernel / D2H
    overlap) or a torch CUDA tensor (device path, current stream).
    Returns a dict of arrays (numpy for host input, torch for device input):
    total, datap, pipelinep and optionally per_group [P, d_pp], order [P, d_pp].
    Malformed partitions raise CostModelError.

    ``devices=[d0, d1, ...]`` splits the population contiguously over those
    GPUs (shard_bounds), each pricing its slice against its own replica of
    the pair tables, concurrently; results are gathered back in input order
    (numpy for host input, a tensor on the input's device otherwise).  This
    is the batch seam the reference parallelises with ``threads``
    (scheduler.py:537-542), bit-identical to one device.
    """
    validate_workload(w, g.lat.shape[0])
    if devices is not None and len(devices) > 1:
        return _comm_cost_batch_multi(g, groups, w, per_group, order, heuristic, [int(d) for d in devices])
    if devices is not None and len(devices) == 1:
        device = int(devices[0])
    if w.d_pp > 16:
        if not heuristic:
            raise ValueError(f"exact path search is limited to 16 vertices, got {w.d_pp}; "
                             "pass heuristic=True to accept an approximate tour")
        return _comm_cost_batch_heuristic(g, groups, w, per_group, order, device)
    inst = N.instance_for(g, w, device)
    k = inst.k
    if isinstance(groups, np.ndarray) or not hasattr(groups, "data_ptr"):
        a = np.ascontiguousarray(groups, dtype=np.int16)
        if a.ndim != 3 or a.shape[1:] != (inst.k, inst.m):
            raise CostModelError(f"expected groups of shape [P, {inst.k}, {inst.m}], got {a.shape}")
        P = a.shape[0]
        out = _host_outputs(P, k, per_group, order)
        nbad = _eval_host_into(inst, a, out)
    else:
        torch = N.torch_cuda()
        t = groups
        if t.dtype != torch.int16 or not t.is_contiguous() or t.device.index != inst.device:
            t = t.to(device=f"cuda:{inst.device}", dtype=torch.int16).contiguous()
        if t.dim() != 3 or tuple(t.shape[1:]) != (inst.k, inst.m):
            raise CostModelError(f"expected groups of shape [P, {inst.k}, {inst.m}], got {tuple(t.shape)}")
        P = t.shape[0]
        out, bad = _launch_device(inst, t, per_group, order)
        nbad = int(bad.item())
    if nbad:
        raise CostModelError(
            f"{nbad} of {P} partitions are not balanced partitions of 0..N-1 with ascending members")
    return out


def _launch_device(inst, t, per_group: bool, order: bool):
    """hs_eval_batch on the device's current stream (no synchronisation):
    returns the output tensors and the device-side malformed-row counter."""
    torch = N.torch_cuda()
    P, k = t.shape[0], inst.k
    dev = f"cuda:{inst.device}"
    out = {name: torch.empty(P, dtype=torch.float64, device=dev) for name in ("total", "datap", "pipelinep")}
    if per_group:
        out["per_group"] = torch.empty((P, k), dtype=torch.float64, device=dev)
    if order:
        out["order"] = torch.empty((P, k), dtype=torch.int8, device=dev)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    N.check(N.lib().hs_eval_batch(inst.handle, t.data_ptr(), P, out["total"].data_ptr(), out["datap"].data_ptr(),
                                  out["pipelinep"].data_ptr(), N.ptr(out.get("per_group")), N.ptr(out.get("order")),
                                  bad.data_ptr(), N.stream_ptr(inst.device)), "hs_eval_batch")
    return out, bad


def _host_outputs(P: int, k: int, per_group: bool, order: bool) -> dict:
    out = {"total": np.empty(P), "datap": np.empty(P), "pipelinep": np.empty(P)}
    if per_group:
        out["per_group"] = np.empty((P, k))
    if order:
        out["order"] = np.empty((P, k), dtype=np.int8)
    return out


def _eval_host_into(inst, a: np.ndarray, out: dict) -> int:
    """hs_eval_batch_host over contiguous host rows ``a`` into the (views
    of) output arrays ``out``; returns the malformed-row count."""
    bad = np.zeros(1, dtype=np.int32)
    N.check(N.lib().hs_eval_batch_host(inst.handle, a.ctypes.data, a.shape[0], N.ptr(out["total"]),
                                       N.ptr(out["datap"]), N.ptr(out["pipelinep"]), N.ptr(out.get("per_group")),
                                       N.ptr(out.get("order")), bad.ctypes.data), "hs_eval_batch_host")
    return int(bad[0])


def _comm_cost_batch_multi(g, groups, w, per_group, order, heuristic, devices):
    """comm_cost_batch over several GPUs: contiguous shards, one replica of
    the pair tables per device, all devices busy at once (host input: one
    host thread per device in the synchronous host-buffer entry, which
    releases the GIL; device input: per-device async launches on each
    device's current stream)."""
    if w.d_pp > 16:
        if not heuristic:
            raise ValueError(f"exact path search is limited to 16 vertices, got {w.d_pp}; "
                             "pass heuristic=True to accept an approximate tour")
    k, m = w.d_pp, w.d_dp
    host = isinstance(groups, np.ndarray) or not hasattr(groups, "data_ptr")
    shape = tuple(groups.shape) if not host else np.shape(groups)
    if len(shape) != 3 or tuple(shape[1:]) != (k, m):
        raise CostModelError(f"expected groups of shape [P, {k}, {m}], got {tuple(shape)}")
    P = shape[0]
    bounds = shard_bounds(P, len(devices))
    if host:
        a = np.ascontiguousarray(groups, dtype=np.int16)
        if w.d_pp > 16:  # the heuristic path returns fresh arrays per shard
            parts = [comm_cost_batch(g, a[lo:hi], w, per_group=per_group, order=order, device=d, heuristic=True)
                     for d, (lo, hi) in zip(devices, bounds)]
            return {key: np.concatenate([p[key] for p in parts]) for key in parts[0]}
        out = _host_outputs(P, k, per_group, order)
        insts = [N.instance_for(g, w, d) for d in devices]  # tables built up front, in order
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=len(devices)) as ex:
            futs = [ex.submit(_eval_host_into, inst, a[lo:hi], {key: val[lo:hi] for key, val in out.items()})
                    for inst, (lo, hi) in zip(insts, bounds) if hi > lo]
            nbad = sum(f.result() for f in futs)
        if nbad:
            raise CostModelError(
                f"{nbad} of {P} partitions are not balanced partitions of 0..N-1 with ascending members")
        return out
    torch = N.torch_cuda()
    src = groups.device
    if w.d_pp > 16:
        parts = [comm_cost_batch(g, groups[lo:hi].cpu().numpy(), w, per_group=per_group, order=order, device=d,
                                 heuristic=True) for d, (lo, hi) in zip(devices, bounds)]
        return {key: torch.from_numpy(np.concatenate([p[key] for p in parts])).to(src) for key in parts[0]}
    shards = []
    for d, (lo, hi) in zip(devices, bounds):  # launch every shard before any synchronisation
        inst = N.instance_for(g, w, d)
        with torch.cuda.device(d):
            t = groups[lo:hi].to(device=f"cuda:{d}", dtype=torch.int16).contiguous()
            shards.append(_launch_device(inst, t, per_group, order))
    nbad = sum(int(bad.item()) for _, bad in shards)
    if nbad:
        raise CostModelError(
            f"{nbad} of {P} partitions are not balanced partitions of 0..N-1 with ascending members")
    return {key: torch.cat([out[key].to(src) for out, _ in shards]) for key in shards[0][0]}


def _comm_cost_batch_heuristic(g, groups, w, per_group, order, device):
    """d_pp > 16 with heuristic=True: NN + 2-opt stage order on the GPU."""
    a = np.ascontiguousarray(groups, dtype=np.int16)
    k, m = w.d_pp, w.d_dp
    if a.ndim != 3 or a.shape[1:] != (k, m):
        raise CostModelError(f"expected groups of shape [P, {k}, {m}], got {a.shape}")
    srt = np.sort(a.reshape(a.shape[0], -1), axis=1)
    if a.shape[0] and not (np.array_equal(srt, np.broadcast_to(np.arange(k * m), srt.shape))
                           and np.all(np.diff(a, axis=2) > 0)):
        raise CostModelError("partitions must cover 0..N-1 with ascending members")
    inst = N.instance_for(g, w, device)
    torch = N.torch_cuda()
    dev = f"cuda:{inst.device}"
    P = a.shape[0]
    t = torch.from_numpy(a).to(dev)
    out = {name: torch.empty(P, dtype=torch.float64, device=dev) for name in ("total", "datap", "pipelinep")}
    out["per_group"] = torch.empty((P, k), dtype=torch.float64, device=dev)
    out["order"] = torch.empty((P, k), dtype=torch.int8, device=dev)
    N.check(N.lib().hs_eval_batch_ex(inst.handle, t.data_ptr(), P, out["total"].data_ptr(), out["datap"].data_ptr(),
                                     out["pipelinep"].data_ptr(), out["per_group"].data_ptr(),
                                     out["order"].data_ptr(), None, 1, N.stream_ptr(inst.device)), "hs_eval_batch_ex")
    res = {key: val.cpu().numpy() for key, val in out.items()}
    if not per_group:
        res.pop("per_group")
    if not order:
        res.pop("order")
    return res


def comm_cost(g, p, w, heuristic: bool = False) -> CostBreakdown:
    """Full bi-level cost of one balanced partition (costmodel.py:217-229)."""
    validate_workload(w, g.lat.shape[0])
    _check_partition(p, g, w)
    r = comm_cost_batch(g, np.asarray([p.groups], dtype=np.int16), w, per_group=True, order=True,
                        heuristic=heuristic)
    total, datap, pipe = float(r["total"][0]), float(r["datap"][0]), float(r["pipelinep"][0])
    return CostBreakdown(datap=datap, pipelinep=pipe, total=total,
                         per_group_datap=tuple(float(x) for x in r["per_group"][0]),
                         pipeline_order=PathResult(tuple(int(x) for x in r["order"][0]), pipe))


def datap_cost(g, p, w) -> tuple[float, tuple[float, ...]]:
    """Data-parallel level: slowest group and the per-group values."""
    _check_partition(p, g, w)
    validate_workload(w, g.lat.shape[0])
    if w.d_dp == 1:
        per = tuple(0.0 for _ in p.groups)
    else:  # the data-parallel level only: no Held-Karp, any d_pp (costmodel.py:171-175)
        per = tuple(float(x) for x in datap_cost_groups(g, np.asarray(p.groups), w))
    return max(per), per


def datap_cost_group(g, group: Iterable[int], w) -> float:
    """Seconds the slowest member of one data-parallel group spends syncing
    (costmodel.py:154-168), priced on the GPU from the raw lat/bw entries."""
    devs = sorted(int(d) for d in group)
    if len(set(devs)) != len(devs):
        raise CostModelError(f"duplicate device in group {devs}")
    if len(devs) != w.d_dp:
        raise CostModelError(f"group size {len(devs)} does not match d_dp {w.d_dp}")
    if devs and (devs[0] < 0 or devs[-1] >= g.lat.shape[0]):
        raise CostModelError(f"device out of range in group {devs}")
    if len(devs) == 1:
        return 0.0
    return float(datap_cost_groups(g, np.asarray([devs]), w)[0])


def datap_cost_groups(g, groups, w) -> np.ndarray:
    """datap_cost_group of each row of int [G, d_dp] (members ascending)."""
    idx = np.asarray(groups, dtype=np.int64)
    G, m = idx.shape
    if m > 128:
        raise CostModelError(f"GPU datap pricing supports groups of <= 128 devices, got {m}")
    if G == 0:
        return np.empty(0)
    lat = np.ascontiguousarray(np.asarray(g.lat)[idx[:, :, None], idx[:, None, :]])
    bw = np.ascontiguousarray(np.asarray(g.bw)[idx[:, :, None], idx[:, None, :]])
    torch = N.torch_cuda()
    dev = N.current_device()
    tl = torch.from_numpy(lat).to(f"cuda:{dev}")
    tb = torch.from_numpy(bw).to(f"cuda:{dev}")
    out = torch.empty(G, dtype=torch.float64, device=f"cuda:{dev}")
    dp_num = float(8.0 * w.c_dp)
    N.check(N.lib().hs_datap_group_batch(tl.data_ptr(), tb.data_ptr(), m, G, float(w.d_dp), dp_num, out.data_ptr(),
                                         dev, N.stream_ptr(dev)), "hs_datap_group_batch")
    return out.cpu().numpy()


def coarsen(g, p, w) -> CoarsenedGraph:
    """Collapse each group to a vertex; edges carry the bottleneck matching
    (costmodel.py:186-197).  The C(k,2) pair matrices are gathered from the
    GPU-built PP table and solved in one batched launch."""
    _check_partition(p, g, w)
    k = len(p.groups)
    pp = N.instance_for(g, w).tables()[1]
    pairs = [(j, j2) for j in range(k) for j2 in range(j + 1, k)]
    grp = [np.asarray(gr, dtype=np.int64) for gr in p.groups]
    edge = np.zeros((k, k))
    matchings: dict = {}
    if pairs:
        stack = np.stack([pp[np.ix_(grp[j], grp[j2])] for j, j2 in pairs])
        vals, prs = bottleneck_matchings(stack)
        for (j, j2), v, pr in zip(pairs, vals, prs):
            edge[j, j2] = edge[j2, j] = v
            matchings[(j, j2)] = MatchingResult(tuple(int(x) for x in pr), float(v))
    return CoarsenedGraph(edge, matchings)


def pipeline_cost(cg, heuristic: bool = False) -> tuple[float, PathResult]:
    """Cheapest open chain through a coarsened edge matrix (costmodel.py:211-214)."""
    res = open_loop_tsp(cg.edge_cost if hasattr(cg, "edge_cost") else cg, heuristic=heuristic)
    return res.total, res


MAX_BRUTE_FORCE_DEVICES = 8


def brute_force_best(g, w, max_devices: int = MAX_BRUTE_FORCE_DEVICES, chunk: int = 1 << 20):
    """Exhaustive optimum over all balanced partitions (costmodel.py:246-266).

    Candidates are unranked on the GPU in the reference's enumeration order
    (lexicographic canonical keys) and priced in bulk; ties keep the first,
    i.e. the lexicographically smallest key.  ``max_devices`` defaults to the
    reference's limit of 8; raise it (e.g. 16) for ground-truth optima the
    reference cannot afford."""
    validate_workload(w, g.lat.shape[0])
    n = g.lat.shape[0]
    if n > max_devices:
        raise CostModelError(f"exhaustive search is limited to {max_devices} devices, got {n}")
    if w.d_pp > 16:
        raise CostModelError("exhaustive search needs exact pricing (d_pp <= 16)")
    torch = N.torch_cuda()
    inst = N.instance_for(g, w)
    dev = f"cuda:{inst.device}"
    total = int(N.lib().hs_count_partitions(n, w.d_dp))
    best_t, best_i = None, -1
    for start in range(0, total, chunk):
        cnt = min(chunk, total - start)
        parts = torch.empty((cnt, w.d_pp, w.d_dp), dtype=torch.int16, device=dev)
        N.check(N.lib().hs_unrank_partitions(n, w.d_pp, w.d_dp, start, cnt, parts.data_ptr(),
                                             N.stream_ptr(inst.device)), "hs_unrank_partitions")
        tot = comm_cost_batch(g, parts, w)["total"].cpu().numpy()
        i = int(np.argmin(tot))  # first minimum
        if best_t is None or tot[i] < best_t:
            best_t, best_i = tot[i], start + i
    one = torch.empty((1, w.d_pp, w.d_dp), dtype=torch.int16, device=dev)
    N.check(N.lib().hs_unrank_partitions(n, w.d_pp, w.d_dp, best_i, 1, one.data_ptr(), N.stream_ptr(inst.device)),
            "hs_unrank_partitions")
    p = Partition.from_groups(one.cpu().numpy()[0].tolist())
    return p, comm_cost(g, p, w)
