"""CLI parity that needs no GPU: profile generation (host input formats) and
every validation / usage / file-system exit path, against the reference's
recorded outputs (tests/golden/cli)."""
from __future__ import annotations

import pytest

from tests import _cli_replay as R

DATA = R.load()


@pytest.mark.parametrize("name", ["gen_case5", "gen_case2_seed", "gen_custom"])
def test_scenario_gen_byte_identical(name, tmp_path, monkeypatch, capsys):
    c = R.case(DATA, name)
    monkeypatch.chdir(tmp_path)
    R.stage(DATA, tmp_path)
    for f in c["outputs"]:
        (tmp_path / f).unlink()
    rc, out, err = R.run(c["argv"], capsys)
    assert (rc, out, err) == (c["rc"], c["stdout"], c["stderr"])
    for f, want in c["outputs"].items():
        assert R.normalize((tmp_path / f).read_text()) == R.normalize(want)


@pytest.mark.parametrize("name", ["gen_custom_nospec", "missing_file", "workload_mismatch", "eval_bad_grid"])
def test_error_paths(name, tmp_path, monkeypatch, capsys):
    c = R.case(DATA, name)
    monkeypatch.chdir(tmp_path)
    R.stage(DATA, tmp_path)
    rc, out, err = R.run(c["argv"], capsys)
    assert rc == c["rc"]
    assert out == c["stdout"]
    assert err == c["stderr"]


def test_usage_error_exit_code(tmp_path, monkeypatch, capsys):
    c = R.case(DATA, "bad_pop")
    monkeypatch.chdir(tmp_path)
    R.stage(DATA, tmp_path)
    rc, _, err = R.run(c["argv"], capsys)
    assert rc == c["rc"] == 2
    # same argparse complaint (the usage line also lists --backend)
    assert err.strip().splitlines()[-1] == c["stderr"].strip().splitlines()[-1]


def test_backend_flag_not_echoed():
    from paper_2206_01288_b200.cli import _echo
    assert _echo(["schedule", "--backend", "gpu", "--pop", "4"]) == ["schedule", "--pop", "4"]
    assert _echo(["eval", "--backend=gpu"]) == ["eval"]


def test_profile_roundtrip_and_workloads(tmp_path):
    import numpy as np

    from paper_2206_01288_b200 import netmodel as nm
    from paper_2206_01288_b200 import workload as wl
    prof = nm.generate_scenario(nm.scenario_case(5))
    nm.save_profile(prof, tmp_path / "p.json")
    back = nm.load_profile(tmp_path / "p.json")
    # file units (ms, Gbit/s) round-trip to within an ulp, as in the reference
    assert np.allclose(back.delay, prof.delay, rtol=1e-15, atol=0)
    assert np.allclose(back.bandwidth, prof.bandwidth, rtol=1e-15, atol=0)
    assert back.names == prof.names
    assert np.array_equal(nm.symmetrize(prof).lat, nm.scenario_case(5).graph().lat)
    (tmp_path / "w.json").write_text(DATA["inputs"]["workload.json"])
    w = wl.load_workload(tmp_path / "w.json")
    assert (w.d_pp, w.d_dp, w.c_pp, w.c_dp) == (8, 8, 1073741824.0, 301989888.0)
    d = wl.workload_from_dict(DATA_JSON("workload_derived.json"))
    assert (d.d_pp, d.d_dp, d.c_pp, d.c_dp) == (2, 4, 2147483648.0, 1207959552.0)
    with pytest.raises(wl.WorkloadError, match="missing key"):
        wl.workload_from_dict({"d_pp": 2})
    with pytest.raises(nm.ProfileError, match="missing key 'delay_ms'"):
        nm.profile_from_dict({"devices": 2})


def DATA_JSON(name):
    import json
    return json.loads(DATA["inputs"][name])


# hetsched/__init__.py:11-70, the reference's public surface
REFERENCE_EXPORTS = """CommGraph NetworkProfile ScenarioSpec edge_cost generate_scenario load_profile save_profile
scenario_case symmetrize ModelSpec ParallelSpec WorkloadSpec derive_workload load_workload validate_workload
MatchingResult PathResult bottleneck_perfect_matching bottleneck_value brute_force_bottleneck_matching
brute_force_open_loop_tsp open_loop_tsp path_cost CoarsenedGraph CostBreakdown Partition brute_force_best coarsen
comm_cost datap_cost datap_cost_group pipeline_cost ScheduleConfig ScheduleResult SurrogateWeights crossover evolve
gain_kl gain_ours init_population local_search Assignment ComparisonReport compare_baselines evaluate_assignment
materialize random_assignment validate_assignment""".split()


def test_reference_public_surface_present():
    import paper_2206_01288_b200 as hs
    assert [n for n in REFERENCE_EXPORTS if not hasattr(hs, n)] == []
