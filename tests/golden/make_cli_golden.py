#!/usr/bin/env python3
"""Record the REFERENCE command line's outputs as CLI parity fixtures.

Run here (the build container), where the reference is importable read-only:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_cli_golden.py

Every case runs `python -m hetsched ...` in a scratch directory holding the
input files under fixed relative names, and stores the inputs, the files the
command wrote, its stdout/stderr and exit code under tests/golden/cli/.
tests/test_cli_cpu.py and tests/test_gpu_cli.py replay the same argv through
paper_2206_01288_b200.cli and compare byte for byte, except the manifest's
duration_s (the one field the reference itself says varies, cli.py:1-10).
"""
from __future__ import annotations

import json
import os
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

OUT = Path(__file__).resolve().parent / "cli"

SPEC = {"case": "three_sites", "groups": [{"size": 4, "delay_ms": 0.2, "bw_gbps": 40, "label": "a"},
                                           {"size": 2, "delay_ms": 1.5, "bw_gbps": 10},
                                           {"size": 2, "delay_ms": 0.5, "bw_gbps": 25, "label": "c"}],
        "cross": {"delay_ms": [5, 40], "bw_gbps": [0.5, 2.0]}, "seed": 11}
WORKLOAD = {"d_pp": 8, "d_dp": 8, "c_pp_bytes": 1073741824, "c_dp_bytes": 301989888}
WORKLOAD_DERIVED = {"model": {"layers": 24, "hidden": 2048, "seq_len": 2048},
                    "parallel": {"d_pp": 2, "d_dp": 4, "global_batch": 1024}}
WORKLOAD_BAD = {"d_pp": 4, "d_dp": 4, "c_pp_bytes": 1, "c_dp_bytes": 1}

# (name, argv, files the command writes)
CASES = [
    ("gen_case5", ["scenario", "gen", "--case", "5", "--out", "profile5.json"], ["profile5.json"]),
    ("gen_case2_seed", ["scenario", "gen", "--case", "2", "--seed", "4", "--out", "profile2.json"], ["profile2.json"]),
    ("gen_custom", ["scenario", "gen", "--case", "custom", "--spec", "spec.json", "--seed", "3", "--out",
                    "profile8.json"], ["profile8.json"]),
    ("gen_custom_nospec", ["scenario", "gen", "--case", "custom", "--out", "x.json"], []),
    ("schedule_ours", ["schedule", "--scenario", "profile5.json", "--workload", "workload.json", "--pop", "16",
                       "--gens", "40", "--seed", "1", "--out", "sched.json", "--trace", "trace.csv"],
     ["sched.json", "trace.csv"]),
    ("schedule_kl_patience", ["schedule", "--scenario", "profile5.json", "--workload", "workload.json", "--pop", "8",
                              "--gens", "60", "--seed", "2", "--local-search", "kl", "--patience", "5", "--out",
                              "sched_kl.json"], ["sched_kl.json"]),
    ("schedule_small", ["schedule", "--scenario", "profile8.json", "--workload", "workload_derived.json", "--pop",
                        "6", "--gens", "25", "--seed", "5", "--max-passes", "3", "--local-search", "none", "--out",
                        "sched8.json", "--trace", "trace8.csv"], ["sched8.json", "trace8.csv"]),
    ("eval_full", ["eval", "--scenario", "profile5.json", "--workload", "workload.json", "--assignment",
                   "assign_full.json"], []),
    ("eval_grid_only", ["eval", "--scenario", "profile5.json", "--workload", "workload.json", "--assignment",
                        "assign_grid.json"], []),
    ("eval_bad_grid", ["eval", "--scenario", "profile5.json", "--workload", "workload.json", "--assignment",
                       "assign_bad.json"], []),
    ("compare", ["compare", "--scenario", "profile5.json", "--workload", "workload.json", "--pop", "8", "--gens",
                 "10", "--seed", "3", "--random-trials", "25", "--out", "cmp.json"], ["cmp.json"]),
    ("missing_file", ["schedule", "--scenario", "nope.json", "--workload", "workload.json", "--out", "o.json"], []),
    ("workload_mismatch", ["schedule", "--scenario", "profile5.json", "--workload", "workload_bad.json", "--out",
                           "o.json"], []),
    ("bad_pop", ["schedule", "--scenario", "profile5.json", "--workload", "workload.json", "--pop", "1", "--out",
                 "o.json"], []),
]


def _assignments(work: Path) -> None:
    """A materialized layout of a random partition (full provenance), its
    bare grid, and a grid with a duplicated device."""
    sys.path.insert(0, os.environ.get("PYTHONPATH", ""))
    import numpy as np
    import hetsched as H
    from hetsched import scheduler as S
    prof = H.load_profile(work / "profile5.json")
    g = H.symmetrize(prof)
    w = H.WorkloadSpec(8, 8, 1073741824, 301989888)
    p = S.random_partition(np.random.Generator(np.random.PCG64(9)), 64, 8, 8)
    a = H.materialize(g, p, w)
    (work / "assign_full.json").write_text(json.dumps(a.to_dict()))
    (work / "assign_grid.json").write_text(json.dumps({"grid": [list(r) for r in a.grid]}))
    bad = [list(r) for r in a.grid]
    bad[0][0] = bad[0][1]
    (work / "assign_bad.json").write_text(json.dumps({"grid": bad}))


def main() -> None:
    if OUT.exists():
        shutil.rmtree(OUT)
    OUT.mkdir(parents=True)
    work = Path(tempfile.mkdtemp(prefix="hs_cli_"))
    for name, payload in (("spec.json", SPEC), ("workload.json", WORKLOAD),
                          ("workload_derived.json", WORKLOAD_DERIVED), ("workload_bad.json", WORKLOAD_BAD)):
        (work / name).write_text(json.dumps(payload, indent=2) + "\n")
    cases = []
    for name, argv, outputs in CASES:
        if name == "eval_full":
            _assignments(work)
        r = subprocess.run([sys.executable, "-m", "hetsched", *argv], cwd=work, capture_output=True, text=True)
        rec = {"name": name, "argv": argv, "rc": r.returncode, "stdout": r.stdout, "stderr": r.stderr,
               "outputs": {}}
        for f in outputs:
            rec["outputs"][f] = (work / f).read_text()
        cases.append(rec)
        print(name, r.returncode, r.stdout.strip()[:60], r.stderr.strip()[:80], flush=True)
    inputs = {}
    for f in ("spec.json", "workload.json", "workload_derived.json", "workload_bad.json", "assign_full.json",
              "assign_grid.json", "assign_bad.json"):
        inputs[f] = (work / f).read_text()
    (OUT / "cases.json").write_text(json.dumps({"inputs": inputs, "cases": cases}, indent=1))
    shutil.rmtree(work)


if __name__ == "__main__":
    main()
