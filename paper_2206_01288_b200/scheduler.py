"""Hybrid genetic search over balanced partitions, on the GPU.

Drop-in mirror of hetsched/scheduler.py: ``ScheduleConfig`` (:36-59),
``SurrogateWeights`` (:62-88), ``ScheduleResult`` (:91-111),
``random_partition`` / ``init_population`` (:114-136), ``crossover``
(:139-174), ``gain_ours`` / ``gain_kl`` (:181-230), ``local_search``
(:490-512) and ``evolve`` (:515-574).  The search runs in the sm_100a
library (K2/K3 in csrc/hs_search.cu): one CTA per GA instance, the numpy
PCG64 stream reproduced draw for draw, so results (partition, cost, trace,
evaluations) are bit-identical to the reference for the same seed.
Callers' ``np.random.Generator`` objects are advanced exactly as the
reference would advance them.

``evolve_islands`` is the new capability: many independent instances per
GPU (seeded like ``SeedSequence(seed).spawn``), optionally exchanging elites
every few generations, across GPUs through torch.distributed (NCCL).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .costmodel import CostBreakdown, Partition, _check_partition
from .combinatorics import PathResult
from .workload import validate_workload

LOCAL_SEARCH_KINDS = ("ours", "kl", "none")
_KIND = {"ours": 0, "kl": 1, "none": 2}


class ScheduleError(ValueError):
    """Invalid scheduler configuration or arguments."""


@dataclass(frozen=True)
class ScheduleConfig:
    pop_size: int = 64
    generations: int = 1000
    local_search: str = "ours"
    max_passes: int = 8
    seed: int = 0
    patience: int | None = None

    def __post_init__(self) -> None:
        if self.pop_size < 2:
            raise ScheduleError(f"pop_size must be >= 2, got {self.pop_size}")
        if self.generations < 1:
            raise ScheduleError(f"generations must be >= 1, got {self.generations}")
        if self.max_passes < 1:
            raise ScheduleError(f"max_passes must be >= 1, got {self.max_passes}")
        kind = str(self.local_search).lower()
        if kind not in LOCAL_SEARCH_KINDS:
            raise ScheduleError(f"local_search must be one of {LOCAL_SEARCH_KINDS}, got {self.local_search!r}")
        object.__setattr__(self, "local_search", kind)
        if self.patience is not None and self.patience < 1:
            raise ScheduleError(f"patience must be >= 1 when set, got {self.patience}")


@dataclass(frozen=True, eq=False)
class SurrogateWeights:
    """w[d][d2] = lat + 8*(c_pp + c_dp)/bw, symmetric, zero diagonal."""

    w: np.ndarray

    def __post_init__(self) -> None:
        w = np.array(self.w, dtype=float)
        if w.ndim != 2 or w.shape[0] != w.shape[1]:
            raise ScheduleError(f"surrogate weights must be square, got shape {w.shape}")
        if not np.array_equal(w, w.T):
            raise ScheduleError("surrogate weights must be symmetric")
        if np.any(w < 0) or np.any(np.diagonal(w) != 0):
            raise ScheduleError("surrogate weights must be nonnegative with a zero diagonal")
        w.setflags(write=False)
        object.__setattr__(self, "w", w)

    @classmethod
    def from_instance(cls, g, workload) -> "SurrogateWeights":
        """Built by the K0 kernel (same bits as scheduler.py:84-88)."""
        _, _, sw = N.instance_for(g, workload).tables()
        return cls(sw)


@dataclass(frozen=True)
class ScheduleResult:
    best_partition: Partition
    best_cost: CostBreakdown
    trace: tuple[tuple[int, float, float], ...]
    evaluations: int
    seed: int

    def to_dict(self) -> dict:
        return {
            "partition": [list(grp) for grp in self.best_partition.key()],
            "cost": self.best_cost.to_dict(),
            "trace": [[gen, best, mean] for gen, best, mean in self.trace],
            "evaluations": self.evaluations,
            "seed": self.seed,
        }

    def trace_csv(self) -> str:
        lines = ["generation,best_cost_s,mean_cost_s"]
        lines.extend(f"{gen},{best!r},{mean!r}" for gen, best, mean in self.trace)
        return "\n".join(lines) + "\n"


def _groups(p) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(p.groups if hasattr(p, "groups") else p, dtype=np.int16))


def _states(rngs) -> "C.Array":
    arr = (N.PCG64 * len(rngs))()
    for i, r in enumerate(rngs):
        arr[i] = N.PCG64.from_generator(r)
    return arr


def random_partitions(rng: np.random.Generator, n: int, d_pp: int, d_dp: int, count: int) -> np.ndarray:
    """``count`` sequential random_partition draws as int16 [count, d_pp, d_dp]."""
    if d_pp * d_dp != n:
        raise ScheduleError(f"d_pp*d_dp = {d_pp * d_dp} does not cover {n} devices")
    dev = N.current_device()
    st = _states([rng])
    out = np.empty((count, d_pp, d_dp), dtype=np.int16)
    N.check(N.lib().hs_random_partitions(n, d_pp, d_dp, dev, count, st, out.ctypes.data), "hs_random_partitions")
    st[0].write_back(rng)
    return out


def random_partition(rng: np.random.Generator, n: int, d_pp: int, d_dp: int) -> Partition:
    """Uniform shuffle of device ids chunked into d_pp groups of d_dp."""
    return Partition.from_groups(random_partitions(rng, n, d_pp, d_dp, 1)[0].tolist())


def init_population(g, w, cfg: ScheduleConfig, rng: np.random.Generator | None = None) -> list[Partition]:
    validate_workload(w, g.lat.shape[0])
    if cfg.pop_size < 2:
        raise ScheduleError(f"pop_size must be >= 2, got {cfg.pop_size}")
    if rng is None:
        rng = np.random.Generator(np.random.PCG64(cfg.seed))
    arr = random_partitions(rng, g.lat.shape[0], w.d_pp, w.d_dp, cfg.pop_size)
    return [Partition.from_groups(a.tolist()) for a in arr]


def crossover(p1, p2, rng: np.random.Generator) -> Partition:
    """Inject part of one of p2's groups into the same slot of p1."""
    if len(p1.groups) != len(p2.groups) or len(p1.groups[0]) != len(p2.groups[0]):
        raise ScheduleError(
            f"parents must share a shape, got {len(p1.groups)}x{len(p1.groups[0])} and "
            f"{len(p2.groups)}x{len(p2.groups[0])}")
    a, b = _groups(p1), _groups(p2)
    k, m = a.shape
    st = _states([rng])
    out = np.empty_like(a)
    N.check(N.lib().hs_crossover(k * m, k, m, N.current_device(), 1, a.ctypes.data, b.ctypes.data, st,
                                 out.ctypes.data), "hs_crossover")
    st[0].write_back(rng)
    return Partition.from_groups(out.tolist())


def _sw_array(sw) -> np.ndarray:
    return np.ascontiguousarray(sw.w if hasattr(sw, "w") else sw, dtype=np.float64)


def gain_ours(sw, p, j: int, j2: int, cand) -> float:
    """Predicted improvement of swapping cand's d1 (group j) with d1' (group j2)."""
    d1, d2, d1p, d2p = (int(x) for x in cand)
    if j == j2:
        raise ScheduleError("candidate groups must differ")
    gj, gj2 = p.groups[j], p.groups[j2]
    if d1 == d2 or d1 not in gj or d2 not in gj:
        raise ScheduleError(f"d1={d1}, d2={d2} must be distinct members of group {j}")
    if d1p == d2p or d1p not in gj2 or d2p not in gj2:
        raise ScheduleError(f"d1'={d1p}, d2'={d2p} must be distinct members of group {j2}")
    return _gains(sw, p, 0, [(j, j2, d1, d2, d1p, d2p)])[0]


def gain_kl(sw, p, d: int, d2: int) -> float:
    """Classical cut-weight gain of swapping d and d2 across their groups."""
    jd = jd2 = -1
    for gi, grp in enumerate(p.groups):
        if d in grp:
            jd = gi
        if d2 in grp:
            jd2 = gi
    if jd < 0 or jd2 < 0:
        raise ScheduleError(f"devices {d}, {d2} must belong to the partition")
    if jd == jd2:
        raise ScheduleError(f"devices {d} and {d2} are both in group {jd}")
    return _gains(sw, p, 1, [(int(d), int(d2), jd, jd2, 0, 0)])[0]


def _gains(sw, p, kind: int, queries) -> np.ndarray:
    w = _sw_array(sw)
    g = _groups(p)
    k, m = g.shape
    q = np.ascontiguousarray(queries, dtype=np.int32)
    B = q.shape[0]
    groups = np.ascontiguousarray(np.broadcast_to(g, (B, k, m)))
    out = np.empty(B)
    N.check(N.lib().hs_gains(k * m, k, m, N.current_device(), w.ctypes.data, kind, B, groups.ctypes.data,
                             q.ctypes.data, out.ctypes.data), "hs_gains")
    return out


def refine_pass(g, w, p, kind: str, rng: np.random.Generator, phase: int = 0) -> tuple[bool, Partition]:
    """One _pass_ours (phase) / _pass_kl step on the GPU (scheduler.py:394-449)."""
    inst = N.instance_for(g, w)
    a = _groups(p)
    st = _states([rng])
    out = np.empty_like(a)
    ch = np.zeros(1, dtype=np.int32)
    N.check(N.lib().hs_refine_pass(inst.handle, _KIND[kind], int(phase), 1, a.ctypes.data, st, out.ctypes.data,
                                   ch.ctypes.data), "hs_refine_pass")
    st[0].write_back(rng)
    return bool(ch[0]), Partition.from_groups(out.tolist())


def local_search(g, w, p, kind: str = "ours", rng: np.random.Generator | None = None, max_passes: int = 8) -> Partition:
    """Refine one partition; returns the best true-cost configuration seen."""
    kind = str(kind).lower()
    if kind not in ("ours", "kl"):
        raise ScheduleError(f"kind must be 'ours' or 'kl', got {kind!r}")
    if max_passes < 1:
        raise ScheduleError(f"max_passes must be >= 1, got {max_passes}")
    if rng is None:
        rng = np.random.Generator(np.random.PCG64(0))
    validate_workload(w, g.lat.shape[0])
    _check_partition(p, g, w)
    if kind == "ours" and w.d_pp == 1 and w.d_dp >= 2:
        raise ValueError("zero-size array to reduction operation maximum which has no identity")
    inst = N.instance_for(g, w)
    a = _groups(p)
    st = _states([rng])
    out = np.empty_like(a)
    N.check(N.lib().hs_local_search(inst.handle, _KIND[kind], int(max_passes), 1, a.ctypes.data, st,
                                    out.ctypes.data, None, None), "hs_local_search")
    st[0].write_back(rng)
    return Partition.from_groups(out.tolist())


class GASession:
    """Islands of independent steady-state GAs on one GPU (hs_ga_* C-ABI)."""

    def __init__(self, g, w, cfg: ScheduleConfig, rngs, device: int | None = None, mode: str = "cta"):
        """mode "cta": one CTA per island (lowest latency); "warp": one warp per
        island (throughput; d_pp <= 8).  Both give identical results."""
        validate_workload(w, g.lat.shape[0])
        if cfg.local_search == "ours" and w.d_pp == 1 and w.d_dp >= 2:
            raise ValueError("zero-size array to reduction operation maximum which has no identity")
        self.inst = N.instance_for(g, w, device)
        self.cfg = cfg
        self.rngs = list(rngs)
        self.islands = len(self.rngs)
        L = N.lib()
        self._cfg = N.GAConfig(cfg.pop_size, cfg.generations, _KIND[cfg.local_search], cfg.max_passes,
                               cfg.patience or 0)
        st = _states(self.rngs)
        h = C.c_void_p()
        N.check(L.hs_ga_create_ex(self.inst.handle, C.byref(self._cfg), self.islands, st,
                                  1 if mode == "warp" else 0, C.byref(h)), "hs_ga_create_ex")
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        lib = getattr(N, "_lib", None) if N is not None else None
        if h is not None and lib is not None:
            lib.hs_ga_destroy(h)
            self.handle = None

    @property
    def k(self):
        return self.inst.k

    @property
    def m(self):
        return self.inst.m

    def run(self, until: int, stream=None) -> None:
        N.check(N.lib().hs_ga_run(self.handle, int(until), stream if stream is not None
                                  else N.stream_ptr(self.inst.device)), "hs_ga_run")

    def export_elites(self, elites: int):
        """(groups int16 [I, E, k*m], costs f64 [I, E]) as torch CUDA tensors."""
        torch = N.torch_cuda()
        dev = f"cuda:{self.inst.device}"
        gr = torch.empty((self.islands, elites, self.k * self.m), dtype=torch.int16, device=dev)
        co = torch.empty((self.islands, elites), dtype=torch.float64, device=dev)
        N.check(N.lib().hs_ga_export(self.handle, elites, gr.data_ptr(), co.data_ptr(), N.stream_ptr(self.inst.device)),
                "hs_ga_export")
        return gr, co

    def import_elites(self, groups, costs, src) -> None:
        """Island i receives migrants groups[src[i]] (torch CUDA tensors)."""
        torch = N.torch_cuda()
        s = torch.as_tensor(np.asarray(src, dtype=np.int32), device=f"cuda:{self.inst.device}")
        N.check(N.lib().hs_ga_import(self.handle, groups.shape[1], groups.contiguous().data_ptr(),
                                     costs.contiguous().data_ptr(), s.data_ptr(), N.stream_ptr(self.inst.device)),
                "hs_ga_import")
        torch.cuda.current_stream(self.inst.device).synchronize()

    def results(self, seeds=None) -> list[ScheduleResult]:
        I, k, m, G = self.islands, self.k, self.m, self.cfg.generations
        bg = np.empty((I, k, m), dtype=np.int16)
        b3 = np.empty((I, 3))
        pg = np.empty((I, k))
        order = np.empty((I, k), dtype=np.int8)
        tb = np.empty((I, G))
        tm = np.empty((I, G))
        tl = np.empty(I, dtype=np.int32)
        ev = np.empty(I, dtype=np.int64)
        st = (N.PCG64 * I)()
        N.check(N.lib().hs_ga_result(self.handle, bg.ctypes.data, b3.ctypes.data, pg.ctypes.data, order.ctypes.data,
                                     tb.ctypes.data, tm.ctypes.data, tl.ctypes.data, ev.ctypes.data, st),
                "hs_ga_result")
        for i, r in enumerate(self.rngs):
            st[i].write_back(r)
        out = []
        for i in range(I):
            pipe = float(b3[i, 2])
            cb = CostBreakdown(datap=float(b3[i, 1]), pipelinep=pipe, total=float(b3[i, 0]),
                               per_group_datap=tuple(float(x) for x in pg[i]),
                               pipeline_order=PathResult(tuple(int(x) for x in order[i]), pipe))
            n = int(tl[i])
            trace = tuple((t, float(tb[i, t]), float(tm[i, t])) for t in range(n))
            seed = self.cfg.seed if seeds is None else seeds[i]
            out.append(ScheduleResult(Partition.from_groups(bg[i].tolist()), cb, trace, int(ev[i]), seed))
        return out


def evolve(g, w, cfg: ScheduleConfig, threads: int = 1) -> ScheduleResult:
    """Run the genetic algorithm; deterministic for a fixed cfg.seed.

    ``threads`` is accepted for signature compatibility; it never changes
    results (the reference guarantees the same, scheduler.py:537-541)."""
    validate_workload(w, g.lat.shape[0])
    sess = GASession(g, w, cfg, [np.random.Generator(np.random.PCG64(cfg.seed))])
    sess.run(cfg.generations)
    return sess.results()[0]


def island_seeds(seed: int, islands: int, offset: int = 0) -> list[np.random.Generator]:
    """Island streams: PCG64 of SeedSequence(seed).spawn(...) children, the
    convention of evaluation.py:295-298."""
    children = np.random.SeedSequence(seed).spawn(offset + islands)[offset:]
    return [np.random.Generator(np.random.PCG64(c)) for c in children]


# ---------------------------------------------------------------------------
# island model across GPUs (new capability)

def migration_sources(rank: int, world: int, islands_per_rank: int) -> list[int]:
    """Ring over global island ids: island r*I+i receives from r*I+i-1."""
    total = world * islands_per_rank
    return [(rank * islands_per_rank + i - 1) % total for i in range(islands_per_rank)]


def gather_elites(groups, costs, group=None):
    """All-gather [I, E, k*m] int16 layouts and [I, E] f64 costs over the
    default process group (NCCL on GPUs, gloo on CPU); identity if
    torch.distributed is not initialized.  int16 travels as bytes."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return groups, costs
    world = dist.get_world_size(group)
    gb = groups.contiguous().view(torch.uint8)
    gl = [torch.empty_like(gb) for _ in range(world)]
    cl = [torch.empty_like(costs) for _ in range(world)]
    dist.all_gather(gl, gb, group=group)
    dist.all_gather(cl, costs.contiguous(), group=group)
    return torch.cat(gl).view(torch.int16).view(-1, *groups.shape[1:]), torch.cat(cl)


def evolve_islands(g, w, cfg: ScheduleConfig, islands_per_rank: int, migrate_every: int = 0, elites: int = 2,
                   group=None, mode: str = "warp") -> list[ScheduleResult]:
    """Run islands_per_rank GA instances on this rank's GPU, streams from
    SeedSequence(cfg.seed).spawn(world * islands_per_rank); every
    `migrate_every` generations (0 = never) each island sends its `elites`
    best members to the next island of a global ring (NCCL all-gather)."""
    import torch.distributed as dist
    dist_on = dist.is_available() and dist.is_initialized()
    rank = dist.get_rank(group) if dist_on else 0
    world = dist.get_world_size(group) if dist_on else 1
    I = int(islands_per_rank)
    rngs = island_seeds(cfg.seed, I, offset=rank * I)
    sess = GASession(g, w, cfg, rngs, mode=mode if w.d_pp <= 8 else "cta")
    src = migration_sources(rank, world, I)
    gen = 0
    while gen < cfg.generations:
        nxt = cfg.generations if migrate_every <= 0 else min(cfg.generations, gen + migrate_every)
        sess.run(nxt)
        gen = nxt
        if migrate_every > 0 and gen < cfg.generations:
            gr, co = sess.export_elites(elites)
            all_gr, all_co = gather_elites(gr, co, group)
            sess.import_elites(all_gr, all_co, src)
    seeds = [cfg.seed] * I
    return sess.results(seeds)
