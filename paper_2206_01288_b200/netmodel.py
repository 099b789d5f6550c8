"""Network instances for the cost model: CommGraph plus the five preset
scenarios used as benchmark inputs.

Mirrors the parts of hetsched/netmodel.py the hot path consumes:
``CommGraph`` (netmodel.py:93-119), ``symmetrize`` (:122-129), the preset
block scenarios (``scenario_case``, :219-254) and their generator
(``generate_scenario``, :257-290).  The generator must reproduce the
reference matrices bit for bit (same PCG64 draw order: per unordered
region pair, delay first then bandwidth, row-major), which
tests/test_instances.py checks against the sha256 of the reference's own
arrays; plus the profile / scenario-spec JSON formats the CLI reads and
writes (netmodel.py:296-426).
"""
from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path
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


def _first_bad(mask: np.ndarray) -> tuple[int, int]:
    i, j = np.argwhere(mask)[0]
    return int(i), int(j)


@dataclass(frozen=True, eq=False)
class NetworkProfile:
    """Directed per-pair delay (s) and bandwidth (bit/s) for N devices, as
    loaded from a profile file (netmodel.py:43-90); bandwidth diagonal +inf."""

    delay: np.ndarray
    bandwidth: np.ndarray
    names: tuple[str, ...] | None = None

    def __post_init__(self) -> None:
        d = np.array(self.delay, dtype=float)
        b = np.array(self.bandwidth, dtype=float)
        if d.ndim != 2 or d.shape[0] != d.shape[1]:
            raise ProfileError(f"delay matrix must be square, got shape {d.shape}")
        if b.shape != d.shape:
            raise ProfileError(f"bandwidth shape {b.shape} does not match delay shape {d.shape}")
        for bad, what in ((~np.isfinite(d), "non-finite delay"), (d < 0, "negative delay")):
            if bad.any():
                raise ProfileError("%s at (%d,%d)" % ((what,) + _first_bad(bad)))
        nz = np.nonzero(np.diagonal(d) != 0)[0]
        if nz.size:
            raise ProfileError(f"nonzero delay at ({int(nz[0])},{int(nz[0])})")
        off = ~np.eye(d.shape[0], dtype=bool)
        for bad, what in (((b <= 0) & off, "non-positive bandwidth"), (~np.isfinite(b) & off, "non-finite bandwidth")):
            if bad.any():
                raise ProfileError("%s at (%d,%d)" % ((what,) + _first_bad(bad)))
        np.fill_diagonal(b, np.inf)
        if self.names is not None:
            names = tuple(str(x) for x in self.names)
            if len(names) != d.shape[0]:
                raise ProfileError(f"got {len(names)} names for {d.shape[0]} devices")
            object.__setattr__(self, "names", names)
        object.__setattr__(self, "delay", _readonly(d))
        object.__setattr__(self, "bandwidth", _readonly(b))

    @property
    def n(self) -> int:
        return self.delay.shape[0]


def symmetrize(profile, bandwidth=None) -> CommGraph:
    """Average both directions (netmodel.py:122-129): lat = (d + d.T)/2,
    bw = (b + b.T)/2.  Takes a NetworkProfile, or the two raw matrices."""
    if bandwidth is None:
        d, b = profile.delay, profile.bandwidth
    else:
        d = np.asarray(profile, dtype=np.float64)
        b = np.array(bandwidth, dtype=np.float64)
        np.fill_diagonal(b, np.inf)
    return CommGraph((d + d.T) / 2.0, (b + b.T) / 2.0)


def edge_cost(g: CommGraph, d: int, d2: int, payload_bytes: float) -> float:
    """lat + 8*payload/bw across one edge (netmodel.py:132-140).  A scalar
    convenience on the host; the batch path never calls it."""
    if d == d2:
        raise ValueError(f"edge cost requires two distinct devices, got {d} twice")
    if not (0 <= d < g.n and 0 <= d2 < g.n):
        raise ValueError(f"device index out of range: ({d},{d2}) for n={g.n}")
    if payload_bytes < 0:
        raise ValueError(f"negative payload: {payload_bytes}")
    return float(g.lat[d, d2] + (8.0 * payload_bytes) / g.bw[d, d2])


@dataclass(frozen=True)
class GroupSpec:
    """One region: size devices, intra delay (s), intra bandwidth (bit/s)."""

    size: int
    delay_s: float
    bw_bps: float
    label: str | None = None

    def __post_init__(self) -> None:
        if self.size < 1:
            raise ScenarioError(f"group size must be >= 1, got {self.size}")
        if self.delay_s < 0:
            raise ScenarioError(f"negative intra delay: {self.delay_s}")
        if self.bw_bps <= 0:
            raise ScenarioError(f"non-positive intra bandwidth: {self.bw_bps}")


Region = GroupSpec


def _span(v) -> tuple[float, float]:
    if isinstance(v, (int, float)):
        return float(v), float(v)
    lo, hi = v
    return float(lo), float(hi)


@dataclass(frozen=True)
class ScenarioSpec:
    """Block-structured instance (netmodel.py:160-191): regions plus
    cross-region (min, max) ranges; min == max is a fixed value."""

    case: str
    groups: tuple[GroupSpec, ...]
    cross_delay_s: tuple[float, float]
    cross_bw_bps: tuple[float, float]
    seed: int = 0

    def __post_init__(self) -> None:
        groups = tuple(self.groups)
        if not groups:
            raise ScenarioError("scenario needs at least one group")
        object.__setattr__(self, "groups", groups)
        object.__setattr__(self, "cross_delay_s", _span(self.cross_delay_s))
        object.__setattr__(self, "cross_bw_bps", _span(self.cross_bw_bps))
        (dlo, dhi), (blo, bhi) = self.cross_delay_s, self.cross_bw_bps
        if dlo < 0:
            raise ScenarioError(f"negative cross delay: {dlo}")
        if blo <= 0:
            raise ScenarioError(f"non-positive cross bandwidth: {blo}")
        if dlo > dhi or blo > bhi:
            raise ScenarioError("range minimum exceeds maximum")

    # names used by the rest of this package
    @property
    def name(self) -> str:
        return self.case

    @property
    def regions(self) -> tuple[GroupSpec, ...]:
        return self.groups

    @property
    def n(self) -> int:
        return sum(r.size for r in self.groups)

    def matrices(self) -> tuple[np.ndarray, np.ndarray]:
        """(delay, bandwidth) before symmetrization (netmodel.py:257-285):
        one PCG64(seed) stream, per unordered region pair in row-major
        order, delay drawn before bandwidth, fixed ranges not drawn."""
        n = self.n
        delay = np.zeros((n, n))
        bw = np.ones((n, n))
        cuts = np.cumsum([0] + [r.size for r in self.groups])
        for r, lo, hi in zip(self.groups, cuts[:-1], cuts[1:]):
            delay[lo:hi, lo:hi] = r.delay_s
            bw[lo:hi, lo:hi] = r.bw_bps
        gen = np.random.Generator(np.random.PCG64(self.seed))
        (dlo, dhi), (blo, bhi) = self.cross_delay_s, self.cross_bw_bps
        nr = len(self.groups)
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

    def device_names(self) -> tuple[str, ...]:
        out: list[str] = []
        for i, r in enumerate(self.groups):
            lab = r.label if r.label is not None else f"g{i}"
            out.extend(f"{lab}-{j}" for j in range(r.size))
        return tuple(out)

    def graph(self) -> CommGraph:
        return symmetrize(*self.matrices())


Scenario = ScenarioSpec


def generate_scenario(spec: ScenarioSpec) -> NetworkProfile:
    """Profile of a block spec (netmodel.py:257-290), device names
    '<label>-<j>' (label defaults to g<i>)."""
    d, b = spec.matrices()
    return NetworkProfile(d, b, spec.device_names())


_REGIONS_4 = ("california", "ohio", "oregon", "virginia")
_REGIONS_8 = ("oregon", "virginia", "ohio", "tokyo", "seoul", "london", "frankfurt", "ireland")
CASE_NAMES = ("data_center_on_demand", "data_center_spot", "multi_data_center",
              "regional_geo", "world_geo")


def scenario_case(case: int | str, seed: int = 0) -> ScenarioSpec:
    """The paper's five 64-device scenarios (netmodel.py:219-254)."""
    key = str(case)
    if key in CASE_NAMES:
        key = str(CASE_NAMES.index(key) + 1)
    G = GroupSpec
    if key == "1":
        return ScenarioSpec(CASE_NAMES[0], tuple(G(8, 1e-4, 100e9, f"node{i}") for i in range(8)), (2.5e-4, 2.5e-4),
                            (25e9, 25e9), seed)
    if key == "2":
        regs = tuple(G(4, 1e-4, 100e9, f"quad{i}") for i in range(8)) + tuple(
            G(1, 1e-4, 100e9, f"solo{i}") for i in range(32))
        return ScenarioSpec(CASE_NAMES[1], regs, (2.5e-4, 2.5e-4), (10e9, 10e9), seed)
    if key == "3":
        return ScenarioSpec(CASE_NAMES[2], (G(32, 2.5e-4, 10e9, "org0"), G(32, 2.5e-4, 10e9, "org1")),
                            (0.010, 0.010), (1.12e9, 1.12e9), seed)
    if key == "4":
        return ScenarioSpec(CASE_NAMES[3], tuple(G(16, 0.005, 2e9, r) for r in _REGIONS_4), (0.010, 0.070),
                            (1.0e9, 1.3e9), seed)
    if key == "5":
        return ScenarioSpec(CASE_NAMES[4], tuple(G(8, 0.005, 2e9, r) for r in _REGIONS_8), (0.010, 0.250),
                            (0.3e9, 1.3e9), seed)
    raise ScenarioError(f"unknown case {case!r}; expected 1..5 or one of {CASE_NAMES}")


def scenario_from_ms_gbps(regions: Sequence[tuple[int, float, float]], cross_delay_ms, cross_bw_gbps,
                          seed: int = 0, name: str = "custom") -> ScenarioSpec:
    """Spec in file units (ms, Gbit/s), converted like spec_from_dict
    (netmodel.py:367-401) so e.g. 0.1 ms becomes 0.1/1000.0 exactly."""
    regs = tuple(GroupSpec(int(s), float(d) / 1000.0, float(b) * 1e9) for s, d, b in regions)
    dlo, dhi = _span(cross_delay_ms)
    blo, bhi = _span(cross_bw_gbps)
    return ScenarioSpec(name, regs, (dlo / 1000.0, dhi / 1000.0), (blo * 1e9, bhi * 1e9), int(seed))


# ---------------------------------------------------------------------------
# file formats (netmodel.py:296-426): profiles carry delay_ms / bandwidth_gbps


def profile_to_dict(profile: NetworkProfile) -> dict:
    gbps = (profile.bandwidth / 1e9).copy()
    np.fill_diagonal(gbps, 0.0)
    out: dict = {"devices": profile.n}
    if profile.names is not None:
        out["names"] = list(profile.names)
    out["delay_ms"] = (profile.delay * 1000.0).tolist()
    out["bandwidth_gbps"] = gbps.tolist()
    return out


def profile_from_dict(data) -> NetworkProfile:
    if not isinstance(data, dict):
        raise ProfileError(f"profile JSON must be an object, got {type(data).__name__}")
    for key in ("devices", "delay_ms", "bandwidth_gbps"):
        if key not in data:
            raise ProfileError(f"profile JSON missing key {key!r}")
    try:
        dms = np.array(data["delay_ms"], dtype=float)
        gbps = np.array(data["bandwidth_gbps"], dtype=float)
    except (TypeError, ValueError) as exc:
        raise ProfileError(f"matrix entries must be numbers: {exc}") from None
    if dms.ndim != 2 or dms.shape[0] != dms.shape[1]:
        raise ProfileError(f"delay matrix must be square, got shape {dms.shape}")
    n = int(data["devices"])
    if dms.shape[0] != n:
        raise ProfileError(f"devices={n} but delay matrix is {dms.shape[0]}x{dms.shape[1]}")
    if gbps.shape != dms.shape:
        raise ProfileError(f"bandwidth shape {gbps.shape} does not match delay shape {dms.shape}")
    bw = gbps * 1e9
    np.fill_diagonal(bw, np.inf)
    names = data.get("names")
    return NetworkProfile(dms / 1000.0, bw, None if names is None else tuple(names))


def spec_to_dict(spec: ScenarioSpec) -> dict:
    groups = []
    for r in spec.groups:
        item = {"size": r.size, "delay_ms": r.delay_s * 1000.0, "bw_gbps": r.bw_bps / 1e9}
        if r.label is not None:
            item["label"] = r.label
        groups.append(item)
    (dlo, dhi), (blo, bhi) = spec.cross_delay_s, spec.cross_bw_bps
    return {"case": spec.case, "groups": groups,
            "cross": {"delay_ms": [dlo * 1000.0, dhi * 1000.0], "bw_gbps": [blo / 1e9, bhi / 1e9]},
            "seed": spec.seed}


def spec_from_dict(data) -> ScenarioSpec:
    if not isinstance(data, dict):
        raise ScenarioError(f"scenario spec must be a JSON object, got {type(data).__name__}")
    if not data.get("groups"):
        raise ScenarioError("scenario spec needs a non-empty 'groups' list")
    groups = []
    for item in data["groups"]:
        try:
            groups.append(GroupSpec(int(item["size"]), float(item["delay_ms"]) / 1000.0,
                                    float(item["bw_gbps"]) * 1e9, item.get("label")))
        except KeyError as exc:
            raise ScenarioError(f"group entry missing key {exc}") from None
    cross = data.get("cross")
    if cross is None:
        if len(groups) > 1:
            raise ScenarioError("multi-group spec needs a 'cross' entry")
        cd, cb = (0.0, 0.0), (1.0, 1.0)
    else:
        dlo, dhi = _span(cross["delay_ms"])
        blo, bhi = _span(cross["bw_gbps"])
        cd, cb = (dlo / 1000.0, dhi / 1000.0), (blo * 1e9, bhi * 1e9)
    return ScenarioSpec(str(data.get("case", "custom")), tuple(groups), cd, cb, int(data.get("seed", 0)))


def _read_json(source, err):
    text = source.read() if hasattr(source, "read") else Path(source).read_text()
    if isinstance(text, bytes):
        text = text.decode("utf-8")
    try:
        return json.loads(text)
    except json.JSONDecodeError as exc:
        raise err(f"malformed JSON: {exc}") from None


def _write_json(payload, dest) -> None:
    text = json.dumps(payload, indent=2) + "\n"
    if hasattr(dest, "write"):
        dest.write(text)
    else:
        Path(dest).write_text(text)


def load_profile(source) -> NetworkProfile:
    """Profile from a path or an open JSON file."""
    return profile_from_dict(_read_json(source, ProfileError))


def save_profile(profile: NetworkProfile, dest, extra: dict | None = None) -> None:
    """Write a profile as JSON, merging extra top-level keys (a manifest)."""
    payload = profile_to_dict(profile)
    if extra:
        payload.update(extra)
    _write_json(payload, dest)


def load_scenario_spec(source) -> ScenarioSpec:
    return spec_from_dict(_read_json(source, ScenarioError))


def config1_scenario() -> Scenario:
    """BASELINE config 1: 2 nodes x 4 devices with case-1 link values."""
    return scenario_from_ms_gbps([(4, 0.1, 100)] * 2, 0.25, 25, seed=0, name="config1")


def config4_scenario(seed: int = 0) -> Scenario:
    """BASELINE config 4: 512 devices as 16 world-wide regions of 32 with the
    case-5 link ranges."""
    return ScenarioSpec("config4", (GroupSpec(32, 0.005, 2e9),) * 16, (0.010, 0.250), (0.3e9, 1.3e9), seed)


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
