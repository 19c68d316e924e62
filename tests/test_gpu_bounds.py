"""Out-of-bounds guard: every kernel family runs on slices that sit between two guard bands of
NaN-patterned amplitudes.  A stray write changes a guard word; a stray read pulls a NaN into
the result, which then fails the comparison with the oracle.  (compute-sanitizer is not
available on the GPU pool -- runs under it have left GPUs needing a reset -- so this is the
memcheck substitute, at sizes where every grid-edge and tail path is exercised.)"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import random_state

pytestmark = pytest.mark.gpu

sv = pytest.importorskip("paper_1601_07195_b200")
from oracle import oracle  # noqa: E402

DEV = "cuda:0"
GUARD = 1 << 12
CANARY = np.uint64(0x7FF8DEADBEEF0001)  # a quiet NaN with a payload


class Guarded:
    """A 2^m slice inside [guard | slice | guard] of one allocation."""

    def __init__(self, v: np.ndarray):
        self.n = v.shape[0]
        host = np.empty(GUARD + self.n + GUARD, dtype=np.complex128)
        host.view(np.uint64)[:] = CANARY
        host[GUARD:GUARD + self.n] = v
        self.buf = torch.from_numpy(host).to(DEV)
        self.view = self.buf[GUARD:GUARD + self.n]

    def guards_intact(self) -> bool:
        torch.cuda.synchronize()
        w = torch.view_as_real(self.buf).view(torch.int64).view(-1).cpu().numpy().view(np.uint64)
        return bool(np.all(w[:2 * GUARD] == CANARY) and np.all(w[2 * (GUARD + self.n):] == CANARY))

    def numpy(self):
        torch.cuda.synchronize()
        return self.view.cpu().numpy()


def run_guarded(n, circ, fusion=None, exact=True):
    v = random_state(np.random.default_rng(n * 7 + len(circ)), n)
    g = Guarded(v)
    st = sv.LocalState(sv.Layout(n), g.view)
    sv.run_circuit(st, circ, fusion=fusion)
    want = v.copy()
    oracle.run_circuit(want, circ.gates, threads=8)
    got = g.numpy()
    assert g.guards_intact(), "a kernel wrote outside its slice"
    assert np.all(np.isfinite(got)), "a kernel read outside its slice"
    if exact:
        assert np.array_equal(got, want)
    else:
        assert float(np.max(np.abs(got - want))) <= 1e-12 * np.sqrt(len(circ))


@pytest.mark.parametrize("n", [9, 12, 16])
def test_guarded_per_gate_kernels(n):
    rng = np.random.default_rng(n)
    ops = [sv.GateOp(sv.random_unitary(rng), k) for k in range(n)]
    ops += [sv.GateOp(sv.random_unitary(rng), t, c) for c in range(n) for t in range(n) if c != t and (c + t) % 3 == 0]
    run_guarded(n, sv.Circuit(n, ops))


@pytest.mark.parametrize("n,l_c", [(12, 3), (12, 9), (14, 12), (16, 13)])
def test_guarded_fused_blocks(n, l_c):
    circ = sv.random_circuit(n, 80, np.random.default_rng(l_c), controlled_fraction=0.3)
    circ = sv.Circuit(n, [op for op in circ if op.max_qubit() < l_c] + list(circ.gates))
    run_guarded(n, circ, fusion=sv.FusionConfig(l_c=l_c))


@pytest.mark.parametrize("n", [12, 14, 17])
@pytest.mark.parametrize("exact", [True, False])
def test_guarded_pass_planner(n, exact):
    """Register tiles, multi-target stages (exact), k_dstage / k_dlow (tolerance)."""
    circ = sv.build_qft(n)
    circ.extend(sv.random_circuit(n, 120, np.random.default_rng(n), controlled_fraction=0.5).gates)
    circ.extend(sv.build_iqft(n).gates)
    run_guarded(n, circ, fusion=sv.FusionConfig(l_c=min(12, n), passes=True, exact=exact), exact=exact)


@pytest.mark.parametrize("p", [1, 2])
@pytest.mark.parametrize("mode", ["gates", "passes", "remap", "ce"])
def test_guarded_exchange_kernels(p, mode):
    """Exchange, stage-exchange, swap and copy-engine kernels read and write the partner's
    slice: both slices sit between guard bands."""
    n = 13
    m = n - p
    rng = np.random.default_rng(90 + p)
    v = random_state(rng, n)
    circ = sv.build_qft(n)
    circ.extend(sv.random_circuit(n, 60, np.random.default_rng(p), controlled_fraction=0.5).gates)
    gs = [Guarded(v[r << m:(r + 1) << m]) for r in range(1 << p)]
    sts = [sv.LocalState(sv.Layout(n, p, r), g.view) for r, g in enumerate(gs)]
    fabs = sv.InprocFabric.group(sts, data_plane="ce" if mode == "ce" else "ipc", chunk_amps=1 << 7)
    if mode == "remap":
        sv.run_circuit_remapped(sts, circ, fabs)
    else:
        sv.run_circuit_inproc(sts, circ, fabs, fusion=sv.FusionConfig(l_c=11, passes=True) if mode == "passes" else None)
    want = v.copy()
    oracle.run_circuit(want, circ.gates, threads=8)
    got = np.concatenate([g.numpy() for g in gs])
    assert all(g.guards_intact() for g in gs)
    assert np.array_equal(got, want)
