"""Diagonal gates on global qubits without an exchange.

sv_diag_global / sv_diag_fix must reproduce the exchange -- i.e. the
reference's mix() on (own element, partner element), distributed.py:187-202 --
bit for bit, including the sign of zero: the partner only matters through the
sign bits of its original element where the own product has a zero component.
States salted with exact +-0 components, basis states and zero-signed matrix
entries drive that branch.  Checked against the oracle applied to the full
state (an identical-arithmetic restatement of the reference's kernels).
"""

from __future__ import annotations

import os
import tempfile

import numpy as np
import pytest
import torch

from conftest import random_state
from test_gpu_passes import DEV, bits_equal, with_zeros

pytestmark = pytest.mark.gpu

sv = pytest.importorskip("paper_1601_07195_b200")
from oracle import oracle  # noqa: E402
from paper_1601_07195_b200 import _lib  # noqa: E402


def diag_zoo(rng):
    th = rng.uniform(0, 2 * np.pi)
    nz = complex(-0.0, -0.0)
    return [
        sv.phase_r(int(rng.integers(1, 9))), sv.phase_r(int(rng.integers(1, 9))).dagger(), sv.pauli_z(),
        sv.rotation_z(th), sv.phase_shift(th), sv.GateMatrix([[1j, 0], [0, -1j]]),
        sv.GateMatrix.unchecked(np.array([[1, nz], [complex(0.0, -0.0), -1]])),
        sv.GateMatrix.unchecked(np.array([[np.exp(1j * th), complex(-0.0, 0.0)], [nz, 1j]])),
    ]


def states(rng, n):
    basis = np.zeros(1 << n, dtype=np.complex128)
    basis[int(rng.integers(1 << n))] = 1.0
    return [random_state(rng, n), with_zeros(rng, n, 0.3), basis]


def run_abi(slices, m, t, c_local, q):
    """Every rank's sv_diag_global, then (the fence) every rank's sv_diag_fix."""
    L = _lib.load()
    st = torch.cuda.current_stream().cuda_stream
    nbytes = _lib.diag_sign_bytes(m)
    signs = [torch.empty(nbytes, dtype=torch.uint8, device=DEV) for _ in slices]
    flags = [torch.zeros(1, dtype=torch.int32, device=DEV) for _ in slices]
    bit = t - m
    for r, a in enumerate(slices):
        zero = ((r >> bit) & 1) == 0
        _lib.check(L.sv_diag_global(a.data_ptr(), m, int(zero), c_local, q.qbuf(), signs[r].data_ptr(),
                                    flags[r].data_ptr(), st))
    for r, a in enumerate(slices):
        zero = ((r >> bit) & 1) == 0
        _lib.check(L.sv_diag_fix(a.data_ptr(), m, int(zero), c_local, q.qbuf(), signs[r ^ (1 << bit)].data_ptr(),
                                 flags[r].data_ptr(), st))
    return flags


@pytest.mark.parametrize("n,p", [(6, 1), (9, 2), (12, 1), (14, 3), (17, 2)])
def test_diag_global_matches_exchange_bitwise(n, p):
    m = n - p
    rng = np.random.default_rng(700 + 10 * n + p)
    controls = sorted({c for c in (-1, 0, 1, 4, 5, 6, m - 1) if c < m})
    zero_seen = False
    for v in states(rng, n):
        for q in diag_zoo(rng):
            t = m + int(rng.integers(p))
            c = controls[int(rng.integers(len(controls)))]
            want = v.copy()
            oracle.apply_gate(want, (t, None if c < 0 else c, q.mat))
            slices = [torch.from_numpy(v[r << m:(r + 1) << m].copy()).to(DEV) for r in range(1 << p)]
            flags = run_abi(slices, m, t, c, q)
            torch.cuda.synchronize()
            got = np.concatenate([s.cpu().numpy() for s in slices])
            assert bits_equal(got, want), (n, p, t, c, q)
            zero_seen |= any(int(f.item()) for f in flags)
    assert zero_seen  # the sign-map patch ran


def test_diag_abi_guards():
    L = _lib.load()
    st = torch.cuda.current_stream().cuda_stream
    a = torch.zeros(64, dtype=torch.complex128, device=DEV)
    s = torch.empty(_lib.diag_sign_bytes(6), dtype=torch.uint8, device=DEV)
    f = torch.zeros(1, dtype=torch.int32, device=DEV)
    h = sv.hadamard().qbuf()
    assert L.sv_diag_global(a.data_ptr(), 6, 1, -1, h, s.data_ptr(), f.data_ptr(), st) == _lib.SV_EINVAL
    assert "not diagonal" in L.sv_last_error().decode()
    z = sv.pauli_z().qbuf()
    assert L.sv_diag_global(a.data_ptr(), 6, 1, 6, z, s.data_ptr(), f.data_ptr(), st) == _lib.SV_EINVAL
    assert L.sv_diag_global(a.data_ptr(), 6, 1, -1, z, 0, f.data_ptr(), st) == _lib.SV_EINVAL
    assert L.sv_diag_fix(a.data_ptr(), 6, 1, -1, h, s.data_ptr(), f.data_ptr(), st) == _lib.SV_EINVAL


# --------------------------------------------------- two processes, real IPC


def _diag_worker(rank, world, port, path, n, diag):
    import torch.distributed as dist

    import paper_1601_07195_b200 as svm

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        p = world.bit_length() - 1
        d = dict(np.load(path + ".in.npz"))
        fabric = svm.NvlinkFabric(fence="host", diagonal_local=diag)
        circ = svm.Circuit(n, [svm.GateOp(svm.GateMatrix.unchecked(q.reshape(2, 2)), int(t),
                                          None if c < 0 else int(c)) for t, c, q in zip(d["t"], d["c"], d["q"])])
        st = svm.state_from_global(svm.Layout(n, p, rank), d["init"], device="cuda:0")
        svm.run_circuit(st, circ, fabric)
        full = svm.gather_full_state(st, fabric)
        if rank == 0:
            np.savez(path + ".out.npz", full=full, sent=fabric.sent_bytes, recv=fabric.received_bytes)
        fabric.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_two_process_diagonal_local_matches_exchange(world):
    """NvlinkFabric(diagonal_local=True): QFT + diagonal gates on global targets (cases 2, 5, 6)
    bit-identical to the oracle, with less NVLink payload than the exchange path."""
    import torch.multiprocessing as mp

    from test_gpu_exchange import _free_port

    n = 10
    p = world.bit_length() - 1
    m = n - p
    rng = np.random.default_rng(90 + world)
    init = with_zeros(rng, n, 0.2)
    ops = list(sv.build_qft(n).gates)
    for q in diag_zoo(rng):
        t = m + int(rng.integers(p))
        for c in [None, 0, m - 1, 3] + [g for g in range(m, n) if g != t][:1]:
            ops.append(sv.GateOp(q, t, c))
    circ = sv.Circuit(n, ops)
    want = init.copy()
    oracle.run_circuit(want, circ.gates)
    outs = {}
    with tempfile.TemporaryDirectory() as tmp:
        for diag in (False, True):
            path = os.path.join(tmp, f"diag{int(diag)}")
            np.savez(path + ".in.npz", init=init, t=np.array([o.target for o in circ]),
                     c=np.array([-1 if o.control is None else o.control for o in circ]),
                     q=np.stack([o.gate.mat.reshape(4) for o in circ]))
            mp.spawn(_diag_worker, args=(world, _free_port(), path, n, diag), nprocs=world, join=True)
            outs[diag] = dict(np.load(path + ".out.npz"))
    for diag in (False, True):
        assert bits_equal(outs[diag]["full"], want), diag
    assert 0 < int(outs[True]["sent"]) < int(outs[False]["sent"])
