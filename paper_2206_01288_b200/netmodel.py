"""Network instances for the cost model: CommGraph plus the five preset
scenarios used as benchmark inputs.

Mirrors the parts of hetsched/netmodel.py the hot path consumes:
``CommGraph`` (netmodel.py:93-119), ``symmetrize`` (:122-129), the preset
block scenarios (``scenario_case``, :219-254) and their generator
(``generate_scenario``, :257-290).  The generator must reproduce the
reference matrices bit for bit (same PCG64 draw order: per unordered
region pair, delay first then bandwidth, row-major), which
tests/test_instances.py checks against the sha256 of the reference's own
arrays.  JSON profile I/O is out of scope.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np


class ProfileError(ValueError):
    """Malformed or inconsistent network data."""


class ScenarioError(ValueError):
    """Invalid scenario specification."""


def _readonly(a: np.ndarray) -> np.ndarray:
    a.setflags(write=False)
    return a


@dataclass(frozen=True, eq=False)
class CommGraph:
    """Symmetric latency (s) and bandwidth (bit/s) matrices; bw diagonal = +inf."""

    lat: np.ndarray
    bw: np.ndarray

    def __post_init__(self) -> None:
        lat = np.array(self.lat, dtype=np.float64)
        bw = np.array(self.bw, dtype=np.float64)
        if lat.ndim != 2 or lat.shape[0] != lat.shape[1] or bw.shape != lat.shape:
            raise ProfileError("lat and bw must be square matrices of equal shape")
        if not (np.array_equal(lat, lat.T) and np.array_equal(bw, bw.T)):
            raise ProfileError("lat and bw must be symmetric")
        if np.any(lat < 0) or np.any(np.diagonal(lat) != 0):
            raise ProfileError("lat must be nonnegative with a zero diagonal")
        off = ~np.eye(lat.shape[0], dtype=bool)
        if np.any((bw <= 0) & off) or np.any(~np.isfinite(bw) & off):
            raise ProfileError("bw must be positive and finite off the diagonal")
        np.fill_diagonal(bw, np.inf)
        object.__setattr__(self, "lat", _readonly(lat))
        object.__setattr__(self, "bw", _readonly(bw))

    @property
    def n(self) -> int:
        return self.lat.shape[0]


def symmetrize(delay: np.ndarray, bandwidth: np.ndarray) -> CommGraph:
    """Average both directions, as netmodel.py:122-129 does for a profile."""
    d = np.asarray(delay, dtype=np.float64)
    b = np.array(bandwidth, dtype=np.float64)
    np.fill_diagonal(b, np.inf)
    return CommGraph((d + d.T) / 2.0, (b + b.T) / 2.0)


@dataclass(frozen=True)
class Region:
    size: int
    delay_s: float
    bw_bps: float


@dataclass(frozen=True)
class Scenario:
    """Block-structured instance: regions plus cross-region ranges."""

    name: str
    regions: tuple[Region, ...]
    cross_delay_s: tuple[float, float]
    cross_bw_bps: tuple[float, float]
    seed: int = 0

    @property
    def n(self) -> int:
        return sum(r.size for r in self.regions)

    def matrices(self) -> tuple[np.ndarray, np.ndarray]:
        """(delay, bandwidth) before symmetrization (netmodel.py:257-285)."""
        n = self.n
        delay = np.zeros((n, n))
        bw = np.ones((n, n))
        cuts = np.cumsum([0] + [r.size for r in self.regions])
        for r, lo, hi in zip(self.regions, cuts[:-1], cuts[1:]):
            delay[lo:hi, lo:hi] = r.delay_s
            bw[lo:hi, lo:hi] = r.bw_bps
        gen = np.random.Generator(np.random.PCG64(self.seed))
        (dlo, dhi), (blo, bhi) = self.cross_delay_s, self.cross_bw_bps
        nr = len(self.regions)
        for a in range(nr):
            for b in range(a + 1, nr):
                dv = dlo if dlo == dhi else float(gen.uniform(dlo, dhi))
                bv = blo if blo == bhi else float(gen.uniform(blo, bhi))
                ra = slice(cuts[a], cuts[a + 1])
                rb = slice(cuts[b], cuts[b + 1])
                delay[ra, rb] = delay[rb, ra] = dv
                bw[ra, rb] = bw[rb, ra] = bv
        np.fill_diagonal(delay, 0.0)
        np.fill_diagonal(bw, np.inf)
        return delay, bw

    def graph(self) -> CommGraph:
        return symmetrize(*self.matrices())


CASE_NAMES = ("data_center_on_demand", "data_center_spot", "multi_data_center",
              "regional_geo", "world_geo")


def scenario_case(case: int | str, seed: int = 0) -> Scenario:
    """The paper's five 64-device scenarios (netmodel.py:219-254)."""
    key = str(case)
    if key in CASE_NAMES:
        key = str(CASE_NAMES.index(key) + 1)
    if key == "1":
        return Scenario(CASE_NAMES[0], (Region(8, 1e-4, 100e9),) * 8, (2.5e-4, 2.5e-4), (25e9, 25e9), seed)
    if key == "2":
        regs = (Region(4, 1e-4, 100e9),) * 8 + (Region(1, 1e-4, 100e9),) * 32
        return Scenario(CASE_NAMES[1], regs, (2.5e-4, 2.5e-4), (10e9, 10e9), seed)
    if key == "3":
        return Scenario(CASE_NAMES[2], (Region(32, 2.5e-4, 10e9),) * 2, (0.010, 0.010), (1.12e9, 1.12e9), seed)
    if key == "4":
        return Scenario(CASE_NAMES[3], (Region(16, 0.005, 2e9),) * 4, (0.010, 0.070), (1.0e9, 1.3e9), seed)
    if key == "5":
        return Scenario(CASE_NAMES[4], (Region(8, 0.005, 2e9),) * 8, (0.010, 0.250), (0.3e9, 1.3e9), seed)
    raise ScenarioError(f"unknown case {case!r}; expected 1..5 or one of {CASE_NAMES}")


def scenario_from_ms_gbps(regions: Sequence[tuple[int, float, float]], cross_delay_ms, cross_bw_gbps,
                          seed: int = 0, name: str = "custom") -> Scenario:
    """Spec in file units (ms, Gbit/s), converted like spec_from_dict
    (netmodel.py:367-401) so e.g. 0.1 ms becomes 0.1/1000.0 exactly."""

    def rng_of(v):
        lo, hi = (v, v) if isinstance(v, (int, float)) else v
        return float(lo), float(hi)

    regs = tuple(Region(int(s), float(d) / 1000.0, float(b) * 1e9) for s, d, b in regions)
    dlo, dhi = rng_of(cross_delay_ms)
    blo, bhi = rng_of(cross_bw_gbps)
    return Scenario(name, regs, (dlo / 1000.0, dhi / 1000.0), (blo * 1e9, bhi * 1e9), int(seed))


def config1_scenario() -> Scenario:
    """BASELINE config 1: 2 nodes x 4 devices with case-1 link values."""
    return scenario_from_ms_gbps([(4, 0.1, 100)] * 2, 0.25, 25, seed=0, name="config1")


def config4_scenario(seed: int = 0) -> Scenario:
    """BASELINE config 4: 512 devices as 16 world-wide regions of 32 with the
    case-5 link ranges."""
    return Scenario("config4", (Region(32, 0.005, 2e9),) * 16, (0.010, 0.250), (0.3e9, 1.3e9), seed)


def random_graph(seed: int, n: int, lat_range=(0.001, 0.05), bw_range=(1e9, 1e10)) -> CommGraph:
    """Seeded heterogeneous clique (reference tests/conftest.py:50-60 recipe:
    default_rng(seed), lat drawn before bw)."""
    rng = np.random.default_rng(seed)
    lat = rng.uniform(*lat_range, size=(n, n))
    bw = rng.uniform(*bw_range, size=(n, n))
    lat = (lat + lat.T) / 2.0
    bw = (bw + bw.T) / 2.0
    np.fill_diagonal(lat, 0.0)
    np.fill_diagonal(bw, np.inf)
    return CommGraph(lat, bw)
