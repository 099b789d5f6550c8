"""CPU-only checks of the boundary: the sm_100a library loads here (no GPU
needed to dlopen it), exports every entry point include/*.h declares, and
the Python mirror validates like the reference before any compute call."""
from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2206_01288_b200 as hs
from paper_2206_01288_b200 import _native as N

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        names |= set(re.findall(r"\b(hs_[a-z0-9_]+)\s*\(", text))
    return sorted(names)


def test_library_is_built_for_sm100a():
    assert N.LIB_PATH.exists(), "run __graft_entry__.build() first"
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(N.LIB_PATH))
    syms = declared_symbols()
    assert len(syms) >= 8
    for s in syms:
        assert hasattr(lib, s), s
    assert set(N.EXPORTS) == set(syms)
    assert N.lib().hs_version() == 1


def test_partition_validation_messages():
    with pytest.raises(hs.CostModelError, match="disjoint"):
        hs.Partition(((0, 1), (0, 2)))
    with pytest.raises(hs.CostModelError, match="disjoint"):
        hs.Partition(((0, 1), (2, 4)))
    with pytest.raises(hs.CostModelError, match="unbalanced"):
        hs.Partition(((0, 1), (2,)))
    with pytest.raises(hs.CostModelError):
        hs.Partition(((-1, 0), (1, 2)))
    p = hs.Partition(((3, 2), (1, 0)))
    assert p.groups == ((2, 3), (0, 1)) and p.canonical().groups == ((0, 1), (2, 3))


def test_workload_validation_before_any_device_call():
    from tests._instances import g4
    g = g4()
    with pytest.raises(ValueError, match="devices"):
        hs.comm_cost(g, hs.Partition(((0, 1), (2, 3))), hs.WorkloadSpec(d_pp=2, d_dp=3, c_pp=1.0, c_dp=1.0))
    with pytest.raises(hs.CostModelError, match="shape"):
        hs.comm_cost(g, hs.Partition(((0,), (1,), (2,), (3,))), hs.WorkloadSpec(2, 2, 1.0, 1.0))


def test_solver_input_validation():
    with pytest.raises(ValueError, match="square"):
        hs.bottleneck_value([[1.0, 2.0]])
    with pytest.raises(ValueError, match="finite"):
        hs.bottleneck_value([[np.inf]])
    with pytest.raises(ValueError, match="nonnegative"):
        hs.bottleneck_value([[-1.0]])
    with pytest.raises(ValueError, match="symmetric"):
        hs.open_loop_tsp([[0.0, 1.0], [2.0, 0.0]])
    with pytest.raises(ValueError, match="heuristic=True"):
        hs.open_loop_tsp(np.ones((18, 18)) - np.eye(18))
    assert hs.open_loop_tsp([[0.0]]).order == (0,)
    assert hs.path_cost([[0.0, 1.5], [1.5, 0.0]], (0, 1)) == 1.5


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from tests._instances import g4
    with pytest.raises(N.NativeUnavailable):
        hs.comm_cost(g4(), hs.Partition(((0, 1), (2, 3))), hs.WorkloadSpec(2, 2, 1.25e8, 5e8))


def test_batch_assignment_apis_validate_on_host():
    """Malformed rows are rejected before any device call (the kernels index
    the pair tables by these ids)."""
    import numpy as np

    from paper_2206_01288_b200 import PAPER_WORKLOAD, AssignmentError, scenario_case
    from paper_2206_01288_b200.evaluation import evaluate_assignments, materialize_batch
    g = scenario_case(5).graph()
    good = np.arange(64, dtype=np.int16).reshape(1, 8, 8)
    for bad in (good + 1, np.where(good == 5, 4, good), good[:, ::-1, ::-1].copy()):
        with pytest.raises(AssignmentError):
            materialize_batch(g, bad, PAPER_WORKLOAD)
    with pytest.raises(AssignmentError):
        materialize_batch(g, good.reshape(1, 4, 16), PAPER_WORKLOAD)
    grid = np.arange(64, dtype=np.int16).reshape(1, 8, 8)
    with pytest.raises(AssignmentError, match="1 of 2 grids"):
        evaluate_assignments(g, np.concatenate([grid, np.minimum(grid, 62)]), PAPER_WORKLOAD)
