"""bench.py contract pieces that run without a GPU: the reference arm
prints one JSON line from rank 0 only, with n_gpus = the requested N, both
stand-alone and under torchrun (world 2)."""
from __future__ import annotations

import json
import socket
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
ARGS = ["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--cpu-seconds", "0.3"]


def _lines(out: str):
    return [json.loads(ln) for ln in out.splitlines() if ln.startswith("{")]


def test_reference_arm_standalone_gpus2():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *ARGS], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    (line,) = _lines(r.stdout)
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["e2e"]["h2d_bytes_per_step"] == 0


def test_reference_arm_under_torchrun_world2():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", f"--master-port={port}", str(ROOT / "bench.py"), *ARGS],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    (line,) = _lines(r.stdout)
    assert line["n_gpus"] == 2
