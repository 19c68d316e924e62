"""bench.py's rank fan-out (CPU): `--gpus N` without torchrun launches N ranks itself, and a
WORLD_SIZE that disagrees with --gpus fails loudly (mirror of the reference's run_spmd
rank fan-out, pkg/src/svsim/transport.py:274-310)."""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def test_job_size_follows_gpus_and_world():
    assert bench.job_size(bench.parse([]), env={}) == 1
    assert bench.job_size(bench.parse(["--gpus", "4"]), env={}) == 4
    assert bench.job_size(bench.parse([]), env={"WORLD_SIZE": "8"}) == 8
    assert bench.job_size(bench.parse(["--gpus", "2"]), env={"WORLD_SIZE": "2"}) == 2
    with pytest.raises(SystemExit, match="WORLD_SIZE=2"):
        bench.job_size(bench.parse(["--gpus", "4"]), env={"WORLD_SIZE": "2"})
    with pytest.raises(SystemExit, match="power of two"):
        bench.job_size(bench.parse(["--gpus", "3"]), env={})


def test_launch_command_only_outside_torchrun(monkeypatch):
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    cmd = bench.launch_command(bench.parse(["--gpus", "4", "--steps", "2"]), ["--gpus", "4", "--steps", "2"], 29555)
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd and cmd[-4:] == ["--gpus", "4", "--steps", "2"]
    assert bench.launch_command(bench.parse([]), [], 29555) is None
    monkeypatch.setenv("WORLD_SIZE", "4")
    assert bench.launch_command(bench.parse(["--gpus", "4"]), ["--gpus", "4"], 29555) is None


def _run(args, extra_env=None):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update({"SVB_BENCH_PROBE": "1", "MASTER_ADDR": "127.0.0.1"})
    env.update(extra_env or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                          env=env, timeout=300, cwd=ROOT)


def _probes(stdout):
    out = []
    for ln in stdout.splitlines():
        try:
            d = json.loads(ln)
        except ValueError:
            continue
        if isinstance(d, dict) and d.get("probe"):
            out.append(d)
    return out


def test_gpus_two_self_launches_two_ranks():
    for _ in range(2):  # a rendezvous port race on a busy host is retried once
        res = _run(["--gpus", "2"])
        probes = _probes(res.stdout)
        if res.returncode == 0 and len(probes) == 2:
            break
    assert res.returncode == 0, res.stderr[-2000:]
    assert sorted(p["rank"] for p in probes) == [0, 1]
    assert all(p["world"] == 2 and p["n_qubits"] == 31 and p["global_qubits"] == 1 for p in probes)


def test_world_mismatch_fails_loudly():
    res = _run(["--gpus", "4"], {"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert res.returncode != 0
    assert "WORLD_SIZE=2" in res.stderr
