"""Replay the reference CLI fixtures (tests/golden/cli/cases.json, written
by tests/golden/make_cli_golden.py from the reference's own `hetsched`)
through paper_2206_01288_b200.cli, in-process, in a scratch directory with
the same relative file names."""
from __future__ import annotations

import json
import re
from pathlib import Path

GOLDEN = Path(__file__).resolve().parent / "golden" / "cli" / "cases.json"
_DUR = re.compile(r'"duration_s": [-+0-9.eE]+')


def load():
    return json.loads(GOLDEN.read_text())


def case(data, name):
    return next(c for c in data["cases"] if c["name"] == name)


def normalize(text: str) -> str:
    """Blank the manifest's duration_s, the one field allowed to differ."""
    return _DUR.sub('"duration_s": 0', text)


def stage(data, workdir: Path) -> None:
    """Inputs plus the generated profiles later cases read."""
    for name, text in data["inputs"].items():
        (workdir / name).write_text(text)
    for c in data["cases"]:
        if c["argv"][:2] == ["scenario", "gen"]:
            for f, text in c["outputs"].items():
                (workdir / f).write_text(text)


def run(argv, capsys):
    from paper_2206_01288_b200 import cli
    capsys.readouterr()
    try:
        rc = cli.main(list(argv))
    except SystemExit as exc:  # argparse usage errors
        rc = exc.code
    out = capsys.readouterr()
    return rc, out.out, out.err
