"""Instance recipes shared by the parity tests.

Rebuilds every golden-fixture instance with the repo's own generator
(paper_2206_01288_b200.netmodel), never with the reference; the sha256
recorded by tests/golden/make_golden.py proves the matrices are identical.
"""
from __future__ import annotations

import hashlib
import json
from functools import lru_cache
from pathlib import Path

import numpy as np

from paper_2206_01288_b200.netmodel import (CommGraph, config4_scenario, random_graph, scenario_case,
                                            scenario_from_ms_gbps)
from paper_2206_01288_b200.workload import WorkloadSpec

GOLDEN = Path(__file__).resolve().parent / "golden"


def g4() -> CommGraph:
    lat = np.full((4, 4), 0.05)
    bw = np.full((4, 4), 1e9)
    for a, b in ((0, 1), (2, 3)):
        lat[a, b] = lat[b, a] = 0.001
        bw[a, b] = bw[b, a] = 10e9
    np.fill_diagonal(lat, 0.0)
    np.fill_diagonal(bw, np.inf)
    return CommGraph(lat, bw)


def homogeneous(n: int, lat: float = 0.5, bw: float = 8.0) -> CommGraph:
    a = np.full((n, n), lat)
    b = np.full((n, n), bw)
    np.fill_diagonal(a, 0.0)
    np.fill_diagonal(b, np.inf)
    return CommGraph(a, b)


def build(recipe: dict):
    kind = recipe["kind"]
    if kind == "g4":
        g = g4()
    elif kind == "case":
        g = scenario_case(recipe["case"], seed=recipe.get("seed", 0)).graph()
    elif kind == "spec":
        sp = recipe["spec"]
        regs = [(r["size"], r["delay_ms"], r["bw_gbps"]) for r in sp["groups"]]
        g = scenario_from_ms_gbps(regs, sp["cross"]["delay_ms"], sp["cross"]["bw_gbps"], sp.get("seed", 0)).graph()
    elif kind == "random":
        g = random_graph(recipe["seed"], recipe["n"])
    elif kind == "config4":
        g = config4_scenario().graph()
    else:
        raise ValueError(kind)
    return g, WorkloadSpec(*recipe["w"])


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


@lru_cache(None)
def meta():
    return json.loads((GOLDEN / "instances.json").read_text())["instances"]


@lru_cache(None)
def instance(name: str):
    return build(meta()[name]["recipe"])


@lru_cache(None)
def costs():
    return dict(np.load(GOLDEN / "costs.npz"))


def fixture(name: str):
    return json.loads((GOLDEN / name).read_text())


def fx(h: str) -> float:
    return float.fromhex(h)
