#!/usr/bin/env python3
"""Generate the golden parity fixtures by running the REFERENCE itself.

Run here (the build container), where the reference is importable read-only:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--slow]

It writes tests/golden/*.json / *.npz.  Nothing under tests/ imports the
reference at test time; the GPU box only reads these committed files.

Instances are identified by a recipe plus the sha256 of the reference's own
lat/bw bytes, so tests can prove the repo's scenario generator reproduces
the reference matrices bit for bit (netmodel.py:219-290, conftest.py:26-60).
Floats are stored as float.hex() strings (JSON) or float64 arrays (npz).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

import hetsched as H
from hetsched import scheduler as S
from hetsched.netmodel import spec_from_dict

OUT = Path(__file__).resolve().parent
PINNED = H.WorkloadSpec(d_pp=8, d_dp=8, c_pp=1_073_741_824, c_dp=301_989_888)
W4 = H.WorkloadSpec(d_pp=2, d_dp=2, c_pp=125_000_000, c_dp=500_000_000)
CONFIG1_SPEC = {"groups": [{"size": 4, "delay_ms": 0.1, "bw_gbps": 100}] * 2,
                "cross": {"delay_ms": 0.25, "bw_gbps": 25}, "seed": 0}
CONFIG1_W = H.WorkloadSpec(d_pp=2, d_dp=4, c_pp=2_147_483_648, c_dp=1_207_959_552)


def hx(x: float) -> str:
    return float(x).hex()


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def make_g4():
    lat = np.full((4, 4), 0.05)
    bw = np.full((4, 4), 1e9)
    for a, b in ((0, 1), (2, 3)):
        lat[a, b] = lat[b, a] = 0.001
        bw[a, b] = bw[b, a] = 10e9
    np.fill_diagonal(lat, 0.0)
    np.fill_diagonal(bw, np.inf)
    return H.CommGraph(lat=lat, bw=bw)


def make_random_graph(rng, n, lat_range=(0.001, 0.05), bw_range=(1e9, 1e10)):
    lat = rng.uniform(*lat_range, size=(n, n))
    bw = rng.uniform(*bw_range, size=(n, n))
    lat = (lat + lat.T) / 2.0
    bw = (bw + bw.T) / 2.0
    np.fill_diagonal(lat, 0.0)
    np.fill_diagonal(bw, np.inf)
    return H.CommGraph(lat=lat, bw=bw)


# recipe -> (CommGraph, WorkloadSpec)
def instance(recipe: dict):
    kind = recipe["kind"]
    if kind == "g4":
        g = make_g4()
    elif kind == "case":
        g = H.symmetrize(H.generate_scenario(H.scenario_case(recipe["case"], seed=recipe.get("seed", 0))))
    elif kind == "spec":
        g = H.symmetrize(H.generate_scenario(spec_from_dict(recipe["spec"])))
    elif kind == "random":
        g = make_random_graph(np.random.default_rng(recipe["seed"]), recipe["n"])
    elif kind == "config4":
        spec = H.ScenarioSpec("config4", tuple(H.netmodel.GroupSpec(32, 0.005, 2e9, f"r{i}") for i in range(16)),
                              (0.010, 0.250), (0.3e9, 1.3e9), 0)
        g = H.symmetrize(H.generate_scenario(spec))
    else:
        raise ValueError(kind)
    w = H.WorkloadSpec(*recipe["w"])
    return g, w


def wlist(w):
    return [w.d_pp, w.d_dp, w.c_pp, w.c_dp]


INSTANCES = {
    "g4": {"kind": "g4", "w": wlist(W4)},
    **{f"case{c}": {"kind": "case", "case": c, "seed": 0, "w": wlist(PINNED)} for c in range(1, 6)},
    "config1": {"kind": "spec", "spec": CONFIG1_SPEC, "w": wlist(CONFIG1_W)},
    "r8_4x2": {"kind": "random", "seed": 11, "n": 8, "w": [4, 2, 125_000_000, 500_000_000]},
    "r8_2x4": {"kind": "random", "seed": 12, "n": 8, "w": [2, 4, 2e8, 1e8]},
    "r6_3x2": {"kind": "random", "seed": 13, "n": 6, "w": [3, 2, 125_000_000, 500_000_000]},
    "r12_3x4": {"kind": "random", "seed": 14, "n": 12, "w": [3, 4, 125_000_000, 500_000_000]},
    "r12_4x3": {"kind": "random", "seed": 15, "n": 12, "w": [4, 3, 3e8, 7e7]},
    "r16_4x4": {"kind": "random", "seed": 16, "n": 16, "w": [4, 4, 125_000_000, 500_000_000]},
    "r16_2x8": {"kind": "random", "seed": 17, "n": 16, "w": [2, 8, 1e9, 3e8]},
    "r24_3x8": {"kind": "random", "seed": 18, "n": 24, "w": [3, 8, 1e9, 3e8]},
    "r20_5x4": {"kind": "random", "seed": 19, "n": 20, "w": [5, 4, 1e9, 3e8]},
    "r36_6x6": {"kind": "random", "seed": 20, "n": 36, "w": [6, 6, 1e9, 3e8]},
    "r64_8x8": {"kind": "random", "seed": 21, "n": 64, "w": [8, 8, 1_073_741_824, 301_989_888]},
    "r40_4x10": {"kind": "random", "seed": 22, "n": 40, "w": [4, 10, 1e9, 3e8]},
    "r48_3x16": {"kind": "random", "seed": 23, "n": 48, "w": [3, 16, 1e9, 3e8]},
    "r18_9x2": {"kind": "random", "seed": 24, "n": 18, "w": [9, 2, 1e9, 3e8]},
    "r10_10x1": {"kind": "random", "seed": 25, "n": 10, "w": [10, 1, 1e9, 3e8]},
    "r4_1x4": {"kind": "random", "seed": 26, "n": 4, "w": [1, 4, 1e9, 3e8]},
    "r64_2x32": {"kind": "random", "seed": 27, "n": 64, "w": [2, 32, 1e9, 3e8]},
    "r32_16x2": {"kind": "random", "seed": 28, "n": 32, "w": [16, 2, 1e9, 3e8]},
    "r48_12x4": {"kind": "random", "seed": 29, "n": 48, "w": [12, 4, 1e9, 3e8]},
    "r128_16x8": {"kind": "random", "seed": 30, "n": 128, "w": [16, 8, 1_073_741_824, 301_989_888]},
    "config4": {"kind": "config4", "w": [16, 32, 268_435_456, 201_326_592]},
    "config5": {"kind": "random", "seed": 0, "n": 1024, "w": [16, 64, 268_435_456, 201_326_592]},
}


def partitions_from_seed(seed: int, count: int, n: int, k: int, m: int) -> np.ndarray:
    """Sequential random_partition draws (scheduler.py:114-121), as int16."""
    rng = np.random.Generator(np.random.PCG64(seed))
    out = np.empty((count, k, m), dtype=np.int16)
    for i in range(count):
        p = S.random_partition(rng, n, k, m)
        out[i] = np.array(p.groups, dtype=np.int16)
    return out


def gen_costs():
    meta, arrays = {}, {}
    for name, rec in INSTANCES.items():
        g, w = instance(rec)
        count = 400 if g.n == 64 and name.startswith("case") else 120
        if w.d_pp >= 12:
            count = 4 if g.n >= 512 else 12
        if name == "g4":
            parts = np.array([[[0, 1], [2, 3]], [[0, 2], [1, 3]], [[0, 3], [1, 2]]], dtype=np.int16)
        else:
            parts = partitions_from_seed(1000 + len(meta), count, g.n, w.d_pp, w.d_dp)
        P = parts.shape[0]
        tot = np.empty(P); dp = np.empty(P); pp = np.empty(P)
        pg = np.empty((P, w.d_pp)); order = np.empty((P, w.d_pp), dtype=np.int16)
        for i in range(P):
            cb = H.comm_cost(g, H.Partition(tuple(tuple(int(x) for x in row) for row in parts[i])), w)
            tot[i], dp[i], pp[i] = cb.total, cb.datap, cb.pipelinep
            pg[i] = cb.per_group_datap
            order[i] = cb.pipeline_order.order
        meta[name] = {"recipe": rec, "lat_sha": sha(g.lat), "bw_sha": sha(g.bw),
                      "sw_sha": sha(S.SurrogateWeights.from_instance(g, w).w),
                      "parts_seed": None if name == "g4" else 1000 + len(meta) - 0, "count": P}
        # record the seed actually used
        arrays[f"{name}/parts"] = parts
        arrays[f"{name}/total"] = tot
        arrays[f"{name}/datap"] = dp
        arrays[f"{name}/pipelinep"] = pp
        arrays[f"{name}/per_group"] = pg
        arrays[f"{name}/order"] = order
        print("costs", name, P, flush=True)
    return meta, arrays


def gen_solvers():
    out = {"matching": [], "tsp": [], "tsp_heuristic": []}
    rng = np.random.default_rng(2024)
    for k in range(1, 9):
        for t in range(30):
            if t % 3 == 0:
                w = rng.integers(0, 4, size=(k, k)).astype(float)
            else:
                w = rng.uniform(0, 10, size=(k, k))
            r = H.bottleneck_perfect_matching(w)
            out["matching"].append({"w": [hx(x) for x in w.ravel()], "m": k,
                                    "pairs": list(r.pairs), "value": hx(r.bottleneck)})
    for m in (12, 16, 24, 32):
        for t in range(5):
            w = rng.uniform(0, 10, size=(m, m)) if t % 2 else rng.integers(0, 30, size=(m, m)).astype(float)
            out["matching"].append({"w": [hx(x) for x in w.ravel()], "m": m,
                                    "value": hx(H.bottleneck_value(w)),
                                    "pairs": list(H.bottleneck_perfect_matching(w).pairs)})
    for k in list(range(1, 11)) + [12, 13]:
        for t in range(12 if k <= 10 else 2):
            if t % 4 == 0:
                w = rng.integers(0, 3, size=(k, k)).astype(float)
            else:
                w = rng.uniform(0, 10, size=(k, k))
            w = (w + w.T) / 2.0
            np.fill_diagonal(w, 0.0)
            r = H.open_loop_tsp(w)
            out["tsp"].append({"w": [hx(x) for x in w.ravel()], "k": k,
                               "order": list(r.order), "total": hx(r.total)})
    for k in (17, 18, 20):
        w = rng.uniform(1, 10, size=(k, k))
        w = (w + w.T) / 2.0
        np.fill_diagonal(w, 0.0)
        r = H.open_loop_tsp(w, heuristic=True)
        out["tsp_heuristic"].append({"w": [hx(x) for x in w.ravel()], "k": k,
                                     "order": list(r.order), "total": hx(r.total)})
    return out


def groups_of(p):
    return [list(g) for g in p.groups]


def gen_search():
    """Gains, passes, crossover, local search on small/medium instances."""
    out = {"gains": [], "passes": [], "crossover": [], "local_search": [], "fast_edge": []}
    for name in ("g4", "r8_4x2", "r12_3x4", "r16_4x4", "r24_3x8", "case3", "case5", "r64_8x8", "r20_5x4"):
        g, w = instance(INSTANCES[name])
        sw = S.SurrogateWeights.from_instance(g, w)
        rng = np.random.default_rng(7)
        for t in range(6):
            p = S.random_partition(rng, g.n, w.d_pp, w.d_dp)
            if w.d_pp >= 2:
                j, j2 = 0, w.d_pp - 1
                gj, gj2 = p.groups[j], p.groups[j2]
                cand = (gj[0], gj[-1], gj2[-1], gj2[0]) if w.d_dp >= 2 else None
                if cand:
                    out["gains"].append({"inst": name, "groups": groups_of(p), "kind": "ours",
                                         "args": [j, j2, *map(int, cand)],
                                         "value": hx(H.gain_ours(sw, p, j, j2, cand))})
                out["gains"].append({"inst": name, "groups": groups_of(p), "kind": "kl",
                                     "args": [int(gj[0]), int(gj2[-1])],
                                     "value": hx(H.gain_kl(sw, p, gj[0], gj2[-1]))})
            for grp in p.groups:
                if len(grp) >= 2:
                    out["fast_edge"].append({"inst": name, "grp": list(grp),
                                             "edge": list(S._fast_edge(sw.w, list(grp)))})
            for kind in ("ours", "kl"):
                for phase in (0, 1):
                    if kind == "kl" and phase == 1:
                        continue
                    grs = [list(x) for x in p.groups]
                    prng = np.random.Generator(np.random.PCG64(100 + t))
                    if kind == "ours":
                        ch = S._pass_ours(sw.w, grs, prng, phase=phase)
                    else:
                        ch = S._pass_kl(sw.w, grs)
                    st = prng.bit_generator.state
                    out["passes"].append({"inst": name, "kind": kind, "phase": phase, "seed": 100 + t,
                                          "groups": groups_of(p), "changed": bool(ch), "out": grs,
                                          "rng_after": [str(st["state"]["state"]), st["has_uint32"], st["uinteger"]]})
            q = S.random_partition(rng, g.n, w.d_pp, w.d_dp)
            crng = np.random.Generator(np.random.PCG64(200 + t))
            child = H.crossover(p, q, crng)
            st = crng.bit_generator.state
            out["crossover"].append({"inst": name, "p1": groups_of(p), "p2": groups_of(q), "seed": 200 + t,
                                     "child": groups_of(child),
                                     "rng_after": [str(st["state"]["state"]), st["has_uint32"], st["uinteger"]]})
            if name in ("case5", "r64_8x8") and t >= 2:
                continue
            for kind in ("ours", "kl"):
                lrng = np.random.default_rng(300 + t)
                res = H.local_search(g, w, p, kind=kind, rng=lrng)
                st = lrng.bit_generator.state
                out["local_search"].append({"inst": name, "kind": kind, "seed": 300 + t, "groups": groups_of(p),
                                            "out": groups_of(res),
                                            "rng_after": [str(st["state"]["state"]), st["has_uint32"], st["uinteger"]]})
        print("search", name, flush=True)
    return out


def _evolve_job(args):
    name, pop, gens, kind, seed, patience = args
    g, w = instance(INSTANCES[name])
    cfg = H.ScheduleConfig(pop_size=pop, generations=gens, local_search=kind, seed=seed, patience=patience)
    t0 = time.perf_counter()
    res = H.evolve(g, w, cfg)
    dt = time.perf_counter() - t0
    d = res.to_dict()
    return {"inst": name, "pop": pop, "gens": gens, "kind": kind, "seed": seed, "patience": patience,
            "partition": d["partition"], "total": hx(d["cost"]["total"]), "datap": hx(d["cost"]["datap"]),
            "pipelinep": hx(d["cost"]["pipelinep"]),
            "per_group": [hx(x) for x in d["cost"]["per_group_datap"]], "order": d["cost"]["pipeline_order"],
            "evaluations": d["evaluations"], "trace_best": [hx(r[1]) for r in d["trace"]],
            "trace_mean": [hx(r[2]) for r in d["trace"]],
            "trace_csv_sha": hashlib.sha256(res.trace_csv().encode()).hexdigest(), "wall_s": dt}


EVOLVE_FAST = (
    [("g4", 8, 50, k, s, None) for k in ("ours", "kl", "none") for s in (0, 1, 2)]
    + [("g4", 8, 500, "ours", 0, 5), ("g4", 4, 3, "ours", 0, None), ("g4", 2, 20, "ours", 3, None)]
    + [("r8_4x2", 8, 40, k, 4, None) for k in ("ours", "kl", "none")]
    + [("r8_2x4", 8, 40, k, 5, None) for k in ("ours", "kl")]
    + [("r12_3x4", 8, 30, k, 6, None) for k in ("ours", "kl", "none")]
    + [("r16_4x4", 16, 25, k, 7, None) for k in ("ours", "kl")]
    + [("r20_5x4", 8, 20, "ours", 8, None), ("r36_6x6", 8, 10, "ours", 9, None)]
    + [("config1", 16, 60, k, 0, None) for k in ("ours", "kl", "none")]
    + [(f"case{c}", 16, 20, k, 0, None) for c in (1, 2, 3, 4, 5) for k in ("ours", "kl")]
    + [("case5", 64, 60, "ours", 0, None), ("case4", 32, 100, "ours", 1, None)]
)
EVOLVE_SLOW = [(f"case{c}", 64, 1000, "ours", 0, None) for c in (1, 2, 3, 4, 5)] + [
    ("config1", 64, 1000, "ours", 0, None)]


def gen_assignments():
    out = {"materialize": [], "random": []}
    for name in ("g4", "r8_4x2", "r12_3x4", "case1", "case5", "r24_3x8"):
        g, w = instance(INSTANCES[name])
        rng = np.random.default_rng(31)
        for t in range(5):
            p = S.random_partition(rng, g.n, w.d_pp, w.d_dp)
            a = H.materialize(g, p, w)
            cb = H.evaluate_assignment(g, a, w)
            out["materialize"].append({"inst": name, "groups": groups_of(p), "grid": [list(r) for r in a.grid],
                                       "order": list(a.order), "total": hx(cb.total), "datap": hx(cb.datap),
                                       "pipelinep": hx(cb.pipelinep)})
    for name in ("case5", "case1", "r12_3x4"):
        g, w = instance(INSTANCES[name])
        for child in np.random.SeedSequence(0).spawn(20):
            rng = np.random.default_rng(child)
            st = rng.bit_generator.state
            a = H.random_assignment(rng, g.n, w.d_pp, w.d_dp)
            cb = H.evaluate_assignment(g, a, w)
            out["random"].append({"inst": name, "state0": [str(st["state"]["state"]), str(st["state"]["inc"])],
                                  "grid": [list(r) for r in a.grid], "order": list(a.order),
                                  "total": hx(cb.total)})
    return out


def gen_big():
    """BASELINE config 5 (1024 devices): heuristic pricing at 32 x 32 and one
    pass of each local-search flavour (the gains-only stress)."""
    out = {"heuristic_costs": [], "passes": []}
    g = make_random_graph(np.random.default_rng(0), 1024)
    w = H.WorkloadSpec(32, 32, 268_435_456, 201_326_592)
    rng = np.random.Generator(np.random.PCG64(77))
    sw = S.SurrogateWeights.from_instance(g, w)
    for t in range(2):
        p = S.random_partition(rng, 1024, 32, 32)
        cb = H.comm_cost(g, p, w, heuristic=True)
        out["heuristic_costs"].append({"groups": groups_of(p), "total": hx(cb.total), "datap": hx(cb.datap),
                                       "pipelinep": hx(cb.pipelinep), "order": list(cb.pipeline_order.order)})
        for kind, phase in (("ours", 0), ("ours", 1), ("kl", 0)):
            grs = [list(x) for x in p.groups]
            prng = np.random.Generator(np.random.PCG64(500 + t))
            t0 = time.perf_counter()
            ch = S._pass_ours(sw.w, grs, prng, phase=phase) if kind == "ours" else S._pass_kl(sw.w, grs)
            dt = time.perf_counter() - t0
            st = prng.bit_generator.state
            out["passes"].append({"kind": kind, "phase": phase, "seed": 500 + t, "groups": groups_of(p),
                                  "changed": bool(ch), "out": grs, "seconds": dt,
                                  "rng_after": [str(st["state"]["state"]), st["has_uint32"], st["uinteger"]]})
        print("big", t, flush=True)
    return out


def gen_api():
    """Public single-call surface behind coarsen / datap_cost_group and the
    exhaustive oracles (costmodel.py:154-197, combinatorics.py:192-207,345-361)."""
    out = {"brute_matching": [], "brute_tsp": [], "coarsen": [], "datap_group": []}
    rng = np.random.default_rng(99)
    for k in list(range(1, 9)) + [9, 10]:
        for t in range(4 if k < 9 else 1):
            w = rng.integers(0, 3, size=(k, k)).astype(float) if t % 2 == 0 else rng.uniform(0, 5, size=(k, k))
            r = H.brute_force_bottleneck_matching(w)
            out["brute_matching"].append({"k": k, "w": [hx(x) for x in w.ravel()], "pairs": list(r.pairs),
                                          "value": hx(r.bottleneck)})
            s_ = (w + w.T) / 2.0
            np.fill_diagonal(s_, 0.0)
            r2 = H.brute_force_open_loop_tsp(s_)
            out["brute_tsp"].append({"k": k, "w": [hx(x) for x in s_.ravel()], "order": list(r2.order),
                                     "total": hx(r2.total)})
        print("brute", k, flush=True)
    for name, seed in (("case5", 1), ("r12_3x4", 2), ("r16_4x4", 3), ("r36_6x6", 4), ("config1", 5)):
        g, w = instance(INSTANCES[name])
        prng = np.random.Generator(np.random.PCG64(seed))
        for t in range(3):
            p = S.random_partition(prng, g.n, w.d_pp, w.d_dp)
            cg = H.coarsen(g, p, w)
            out["coarsen"].append({
                "instance": name, "groups": groups_of(p),
                "edge": [hx(x) for x in cg.edge_cost.ravel()],
                "matchings": [[j, j2, list(r.pairs), hx(r.bottleneck)] for (j, j2), r in sorted(cg.matchings.items())]})
            for grp in p.groups:
                out["datap_group"].append({"instance": name, "group": list(grp),
                                           "value": hx(H.datap_cost_group(g, grp, w))})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--slow", action="store_true", help="also run the 1000-generation GA anchors")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    only = set(args.only.split(",")) if args.only else None
    env = {"numpy": np.__version__, "python": sys.version.split()[0], "reference": H.__version__}
    if not only or "costs" in only:
        meta, arrays = gen_costs()
        np.savez_compressed(OUT / "costs.npz", **arrays)
        (OUT / "instances.json").write_text(json.dumps({"env": env, "instances": meta}, indent=1))
    if not only or "solvers" in only:
        (OUT / "solvers.json").write_text(json.dumps(gen_solvers()))
    if not only or "search" in only:
        (OUT / "search.json").write_text(json.dumps(gen_search()))
    if not only or "assign" in only:
        (OUT / "assignments.json").write_text(json.dumps(gen_assignments()))
    if not only or "api" in only:
        (OUT / "api.json").write_text(json.dumps(gen_api()))
    if only and "big" in only:
        (OUT / "big.json").write_text(json.dumps(gen_big()))
    if not only or "evolve" in only:
        jobs = list(EVOLVE_FAST)
        with ProcessPoolExecutor(max_workers=os.cpu_count()) as ex:
            res = list(ex.map(_evolve_job, jobs))
        (OUT / "evolve.json").write_text(json.dumps({"env": env, "runs": res}))
        print("evolve fast done", flush=True)
    if args.slow:
        with ProcessPoolExecutor(max_workers=len(EVOLVE_SLOW)) as ex:
            res = list(ex.map(_evolve_job, EVOLVE_SLOW))
        (OUT / "evolve_1000.json").write_text(json.dumps({"env": env, "runs": res}))
        print("evolve slow done", flush=True)


if __name__ == "__main__":
    main()
