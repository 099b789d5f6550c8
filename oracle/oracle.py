"""ctypes wrapper over oracle/libhs_oracle.so.

TEST INFRASTRUCTURE ONLY: the CPU parity checker for the sm_100a product
path.  Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg.  It restates
/root/reference/pkg/src/hetsched (costmodel.py, combinatorics.py,
scheduler.py, evaluation.py); see hs_oracle.c for the per-function file:line
citations.  Pinned against golden vectors produced by the reference itself
(tests/golden/make_golden.py, tests/test_oracle_golden.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "libhs_oracle.so"

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i16p = np.ctypeslib.ndpointer(np.int16, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")


class PCG64State(C.Structure):
    _fields_ = [("state_hi", C.c_uint64), ("state_lo", C.c_uint64), ("inc_hi", C.c_uint64),
                ("inc_lo", C.c_uint64), ("has_uint32", C.c_int32), ("uinteger", C.c_uint32)]

    @classmethod
    def from_generator(cls, rng: np.random.Generator) -> "PCG64State":
        st = rng.bit_generator.state
        s, inc = st["state"]["state"], st["state"]["inc"]
        M = (1 << 64) - 1
        return cls(s >> 64, s & M, inc >> 64, inc & M, st["has_uint32"], st["uinteger"])

    def write_back(self, rng: np.random.Generator) -> None:
        st = rng.bit_generator.state
        st["state"]["state"] = (self.state_hi << 64) | self.state_lo
        st["has_uint32"] = int(self.has_uint32)
        st["uinteger"] = int(self.uinteger)
        rng.bit_generator.state = st

    def as_tuple(self):
        return ((self.state_hi << 64) | self.state_lo, int(self.has_uint32), int(self.uinteger))


class GACfg(C.Structure):
    _fields_ = [("pop_size", C.c_int), ("generations", C.c_int), ("kind", C.c_int),
                ("max_passes", C.c_int), ("patience", C.c_int)]


def build() -> Path:
    if not LIB.exists() or LIB.stat().st_mtime < (HERE / "hs_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(str(LIB))
        L.orc_create.restype = C.c_void_p
        L.orc_create.argtypes = [C.c_int, _f64p, _f64p, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double]
        L.orc_destroy.argtypes = [C.c_void_p]
        L.orc_tables.argtypes = [C.c_void_p, _f64p, _f64p, _f64p]
        L.orc_comm_cost.argtypes = [C.c_void_p, _i32p, _f64p, _f64p, _i32p]
        L.orc_comm_cost_heuristic.argtypes = [C.c_void_p, _i32p, _f64p, _i32p]
        L.orc_comm_cost_batch.argtypes = [C.c_void_p, _i16p, C.c_int64, _f64p, _f64p, _f64p, C.c_int]
        L.orc_bottleneck_value.restype = C.c_double
        L.orc_bottleneck_value.argtypes = [_f64p, C.c_int]
        L.orc_bottleneck_matching.argtypes = [_f64p, C.c_int, _i32p, C.POINTER(C.c_double)]
        L.orc_open_loop_tsp.argtypes = [_f64p, C.c_int, C.POINTER(C.c_double), _i32p]
        L.orc_open_loop_tsp_heuristic.argtypes = [_f64p, C.c_int, C.POINTER(C.c_double), _i32p]
        P = C.POINTER(PCG64State)
        L.orc_next64.restype = C.c_uint64
        L.orc_next64.argtypes = [P]
        L.orc_integers.restype = C.c_int64
        L.orc_integers.argtypes = [P, C.c_int64, C.c_int64]
        L.orc_permutation.argtypes = [P, C.c_int, _i32p]
        L.orc_choice_noreplace_sorted.argtypes = [P, C.c_int, C.c_int, _i32p]
        L.orc_uniform.restype = C.c_double
        L.orc_uniform.argtypes = [P, C.c_double, C.c_double]
        L.orc_random_partition.argtypes = [P, C.c_int, C.c_int, C.c_int, _i32p]
        L.orc_crossover.argtypes = [_i32p, _i32p, C.c_int, C.c_int, P, _i32p]
        L.orc_gain_ours.restype = C.c_double
        L.orc_gain_ours.argtypes = [C.c_void_p, _i32p] + [C.c_int] * 6
        L.orc_gain_kl.restype = C.c_double
        L.orc_gain_kl.argtypes = [C.c_void_p, _i32p, C.c_int, C.c_int]
        L.orc_fast_edge.argtypes = [C.c_void_p, _i32p, C.c_int, _i32p]
        L.orc_local_search.argtypes = [C.c_void_p, _i32p, C.c_int, P, C.c_int]
        L.orc_pass.argtypes = [C.c_void_p, _i32p, C.c_int, P, C.c_int]
        L.orc_evolve.argtypes = [C.c_void_p, C.POINTER(GACfg), P, _i32p, _f64p, _f64p, _i32p, _f64p, _f64p,
                                 C.POINTER(C.c_int64)]
        L.orc_random_assignment.argtypes = [P, C.c_int, C.c_int, C.c_int, _i32p, _i32p]
        L.orc_evaluate_assignment.argtypes = [C.c_void_p, _i32p, _f64p, _f64p]
        L.orc_materialize.argtypes = [C.c_void_p, _i32p, _i32p, _i32p]
        _lib = L
    return _lib


def scalars(c_pp, c_dp):
    """The three host-formed numerators, with Python's own int/float rules
    (costmodel.py:136,141; scheduler.py:85)."""
    return float(8.0 * c_dp), float(8.0 * c_pp), float(8.0 * (c_pp + c_dp))


class Oracle:
    """CPU oracle bound to one (CommGraph-like, WorkloadSpec-like) instance."""

    def __init__(self, lat, bw, d_pp, d_dp, c_pp, c_dp):
        L = lib()
        self.lat = np.ascontiguousarray(lat, dtype=np.float64)
        self.bw = np.ascontiguousarray(bw, dtype=np.float64)
        self.n = self.lat.shape[0]
        self.k, self.m = int(d_pp), int(d_dp)
        dp_num, pp_num, sw_num = scalars(c_pp, c_dp)
        self._h = L.orc_create(self.n, self.lat, self.bw, self.k, self.m, dp_num, pp_num, sw_num)

    @classmethod
    def of(cls, g, w):
        return cls(g.lat, g.bw, w.d_pp, w.d_dp, w.c_pp, w.c_dp)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.orc_destroy(h)
            self._h = None

    def tables(self):
        n = self.n
        dp, pp, sw = (np.empty((n, n)) for _ in range(3))
        lib().orc_tables(self._h, dp, pp, sw)
        return dp, pp, sw

    def comm_cost(self, groups):
        g = np.ascontiguousarray(groups, dtype=np.int32).reshape(self.k, self.m)
        o3 = np.empty(3)
        pg = np.empty(self.k)
        order = np.empty(self.k, dtype=np.int32)
        rc = lib().orc_comm_cost(self._h, g, o3, pg, order)
        if rc:
            raise ValueError(f"oracle comm_cost failed rc={rc}")
        return o3[0], o3[1], o3[2], pg, order

    def comm_cost_heuristic(self, groups):
        g = np.ascontiguousarray(groups, dtype=np.int32).reshape(self.k, self.m)
        o3 = np.empty(3)
        order = np.empty(self.k, dtype=np.int32)
        if lib().orc_comm_cost_heuristic(self._h, g, o3, order):
            raise ValueError("oracle heuristic comm_cost failed")
        return o3[0], o3[1], o3[2], order

    def comm_cost_batch(self, parts, threads=1):
        parts = np.ascontiguousarray(parts, dtype=np.int16)
        P = parts.shape[0]
        t, d, p = np.empty(P), np.empty(P), np.empty(P)
        rc = lib().orc_comm_cost_batch(self._h, parts, P, t, d, p, int(threads))
        if rc:
            raise ValueError(f"oracle batch failed rc={rc}")
        return t, d, p

    def gain_ours(self, groups, j, j2, d1, d2, d1p, d2p):
        g = np.ascontiguousarray(groups, dtype=np.int32)
        return lib().orc_gain_ours(self._h, g, j, j2, d1, d2, d1p, d2p)

    def gain_kl(self, groups, d, d2):
        g = np.ascontiguousarray(groups, dtype=np.int32)
        return lib().orc_gain_kl(self._h, g, d, d2)

    def fast_edge(self, grp):
        g = np.ascontiguousarray(grp, dtype=np.int32)
        out = np.empty(2, dtype=np.int32)
        lib().orc_fast_edge(self._h, g, len(g), out)
        return int(out[0]), int(out[1])

    def one_pass(self, groups, kind, st: PCG64State, phase=0):
        g = np.ascontiguousarray(groups, dtype=np.int32).copy()
        ch = lib().orc_pass(self._h, g, 0 if kind == "ours" else 1, C.byref(st), phase)
        return bool(ch), g.reshape(self.k, self.m)

    def local_search(self, groups, kind, st: PCG64State, max_passes=8):
        g = np.ascontiguousarray(groups, dtype=np.int32).copy()
        lib().orc_local_search(self._h, g, 0 if kind == "ours" else 1, C.byref(st), max_passes)
        return g.reshape(self.k, self.m)

    def evolve(self, pop_size, generations, kind, seed=0, max_passes=8, patience=None, state=None):
        cfg = GACfg(pop_size, generations, {"ours": 0, "kl": 1, "none": 2}[kind], max_passes,
                    patience if patience else 0)
        st = state if state is not None else PCG64State.from_generator(np.random.Generator(np.random.PCG64(seed)))
        bg = np.empty(self.k * self.m, dtype=np.int32)
        b3, pg = np.empty(3), np.empty(self.k)
        order = np.empty(self.k, dtype=np.int32)
        tb, tm = np.empty(generations), np.empty(generations)
        ev = C.c_int64(0)
        rows = lib().orc_evolve(self._h, C.byref(cfg), C.byref(st), bg, b3, pg, order, tb, tm, C.byref(ev))
        if rows < 0:
            raise ValueError(f"oracle evolve failed rc={rows}")
        return {"partition": bg.reshape(self.k, self.m), "total": b3[0], "datap": b3[1], "pipelinep": b3[2],
                "per_group": pg, "order": order, "trace_best": tb[:rows], "trace_mean": tm[:rows],
                "evaluations": ev.value}

    def evaluate_assignment(self, grid):
        gr = np.ascontiguousarray(grid, dtype=np.int32)
        o3, pc = np.empty(3), np.empty(self.k)
        lib().orc_evaluate_assignment(self._h, gr, o3, pc)
        return o3, pc

    def materialize(self, groups):
        g = np.ascontiguousarray(groups, dtype=np.int32)
        grid = np.empty((self.m, self.k), dtype=np.int32)
        order = np.empty(self.k, dtype=np.int32)
        rc = lib().orc_materialize(self._h, g, grid, order)
        if rc:
            raise ValueError(f"oracle materialize failed rc={rc}")
        return grid, order


def bottleneck_value(w):
    w = np.ascontiguousarray(w, dtype=np.float64)
    return lib().orc_bottleneck_value(w, w.shape[0])


def bottleneck_matching(w):
    w = np.ascontiguousarray(w, dtype=np.float64)
    pairs = np.empty(w.shape[0], dtype=np.int32)
    v = C.c_double()
    if lib().orc_bottleneck_matching(w, w.shape[0], pairs, C.byref(v)):
        raise ValueError("matching failed")
    return tuple(int(x) for x in pairs), v.value


def open_loop_tsp(w, heuristic=False):
    w = np.ascontiguousarray(w, dtype=np.float64)
    k = w.shape[0]
    order = np.empty(k, dtype=np.int32)
    t = C.c_double()
    f = lib().orc_open_loop_tsp_heuristic if heuristic else lib().orc_open_loop_tsp
    if f(w, k, C.byref(t), order):
        raise ValueError("tsp failed")
    return tuple(int(x) for x in order), t.value


def rng_state(seed_or_rng) -> PCG64State:
    rng = seed_or_rng if isinstance(seed_or_rng, np.random.Generator) else np.random.Generator(
        np.random.PCG64(seed_or_rng))
    return PCG64State.from_generator(rng)


def cpu_count() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1
