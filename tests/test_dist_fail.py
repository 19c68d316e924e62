"""Fail-loud exchanges (CPU, 2 gloo ranks): ranks that disagree on the protocol step raise
TransportError within seconds instead of hanging, and mark their slice corrupt -- the
reference's test_mismatched_plans_fail_loudly (pkg/tests/test_distributed.py:218-235;
TransportError on a phase desync or timeout, pkg/src/svsim/transport.py:56-79).

The fences all-reduce (max) every rank's step fingerprint and its negation (tag, gate,
control, the plan's chunking), so a desync is seen by every rank at the same fence."""

from __future__ import annotations

import datetime
import json
import os
import socket
import tempfile
import time
from multiprocessing import shared_memory

import numpy as np
import pytest

from test_dist_gloo import ShmOracleExecutor, ShmState


def _worker(rank, world, port, path, scenario):
    import torch.distributed as dist

    import paper_1601_07195_b200 as sv

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                            timeout=datetime.timedelta(seconds=20))
    n, p = 8, 1
    lay = sv.Layout(n, p, rank)
    m = lay.m
    shm = shared_memory.SharedMemory(create=True, size=16 << m, name=f"svf_{os.getpid()}_{rank}")
    amps = np.ndarray((1 << m,), dtype=np.complex128, buffer=shm.buf)
    amps[:] = np.arange(1 << m) + 1j
    state = ShmState(lay, amps, shm)
    fabric = sv.NvlinkFabric(fence="host", executor=ShmOracleExecutor(), data_plane="nccl")
    half = 1 << (m - 1)
    out = {"rank": rank, "raised": None}
    t0 = time.monotonic()
    try:
        if scenario == "chunk":  # the reference's case: ranks plan different chunkings
            sv.apply_single_distributed(state, n - 1, sv.pauli_x(), fabric,
                                        chunk_amps=half if rank == 0 else half // 2)
        elif scenario == "gate":  # ranks at different gates (controlled vs uncontrolled)
            sv.apply_global(state, n - 1, None if rank == 0 else 0, sv.pauli_x(), fabric)
        elif scenario == "skip":  # rank 1 skips the gate and goes on to its next fence
            if rank == 0:
                sv.apply_single_distributed(state, n - 1, sv.pauli_x(), fabric)
            else:
                fabric.barrier(state)
        else:  # agreement: no error
            sv.apply_single_distributed(state, n - 1, sv.pauli_x(), fabric, chunk_amps=half // 2)
    except sv.TransportError as exc:
        out["raised"] = type(exc).__name__
        out["msg"] = str(exc)[:200]
    except Exception as exc:  # noqa: BLE001 -- recorded, the test asserts on it
        out["raised"] = type(exc).__name__
        out["msg"] = str(exc)[:200]
    out["seconds"] = time.monotonic() - t0
    out["corrupt"] = bool(state.corrupt)
    with open(f"{path}.{rank}.json", "w") as fh:
        json.dump(out, fh)
    del amps
    shm.close()
    shm.unlink()
    try:
        dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        pass


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def run(scenario):
    import torch.multiprocessing as mp

    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "f")
        mp.spawn(_worker, args=(2, _port(), path, scenario), nprocs=2, join=True)
        return [json.load(open(f"{path}.{r}.json")) for r in range(2)]


@pytest.mark.parametrize("scenario", ["chunk", "gate", "skip"])
def test_desync_raises_transport_error_quickly(scenario):
    res = run(scenario)
    for r in res:
        assert r["raised"] == "TransportError", r
        assert r["seconds"] < 10.0, r
        assert "desync" in r["msg"], r
    assert any(r["corrupt"] for r in res)


def test_agreeing_ranks_do_not_raise():
    res = run("ok")
    assert all(r["raised"] is None and not r["corrupt"] for r in res), res
