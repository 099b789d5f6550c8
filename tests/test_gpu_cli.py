"""The command line end to end on the GPU: schedule / eval / compare write
byte-identical JSON / CSV and print the same numbers as the reference CLI
(fixtures recorded by tests/golden/make_cli_golden.py); only the manifest's
duration_s may differ."""
from __future__ import annotations

import pytest

from tests import _cli_replay as R

pytestmark = pytest.mark.gpu

DATA = R.load()


@pytest.mark.parametrize("name", ["schedule_ours", "schedule_kl_patience", "schedule_small", "eval_full",
                                  "eval_grid_only", "compare"])
def test_cli_byte_identical(name, tmp_path, monkeypatch, capsys):
    c = R.case(DATA, name)
    monkeypatch.chdir(tmp_path)
    R.stage(DATA, tmp_path)
    argv = list(c["argv"]) + ["--backend", "gpu"]
    rc, out, err = R.run(argv, capsys)
    assert rc == c["rc"] == 0, err
    assert R.normalize(out) == R.normalize(c["stdout"])
    for f, want in c["outputs"].items():
        assert R.normalize((tmp_path / f).read_text()) == R.normalize(want), f
