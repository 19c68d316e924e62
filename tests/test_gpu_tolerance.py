"""Tolerance-mode fusion (FusionConfig(passes=True, exact=False)) against the oracle.

The mode trades bitwise parity for fewer FP64 operations (merged same-qubit
gates, diagonal gates folded into per-amplitude factors by k_dstage), so the
bar is north_star's: max-abs <= 1e-12 * sqrt(G) against the reference's
arithmetic (oracle/sv_oracle.c, pinned to reference-generated goldens) on the
same seeded state and circuit; on a basis input the transform is also checked
against the closed-form DFT (pkg/src/svsim/oracle.py:73-83).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import random_state

pytestmark = pytest.mark.gpu

sv = pytest.importorskip("paper_1601_07195_b200")
from oracle import oracle  # noqa: E402  (checker only)

DEV = "cuda:0"
TOL = sv.FusionConfig(l_c=12, passes=True, exact=False)


def bound(g):
    return 1e-12 * np.sqrt(g)


def run_both(n, circ, v, fusion=TOL):
    st = sv.state_from_global(sv.Layout(n), v, device=DEV)
    sv.run_circuit(st, circ, fusion=fusion)
    torch.cuda.synchronize()
    want = v.copy()
    oracle.run_circuit(want, circ.gates, threads=8)
    return st.to_numpy(), want


@pytest.mark.parametrize("n", [12, 16, 20, 22])
def test_qft_tolerance_vs_oracle(n):
    v = random_state(np.random.default_rng(n), n)
    circ = sv.build_qft(n)
    got, want = run_both(n, circ, v)
    err = float(np.max(np.abs(got - want)))
    assert err <= bound(len(circ)), err
    assert err > 0.0 or n < 14  # the mode really runs a different arithmetic (stage passes appear from n >= 14)


@pytest.mark.parametrize("n", [14, 20])
def test_iqft_round_trip_tolerance(n):
    v = random_state(np.random.default_rng(3 * n), n)
    circ = sv.build_qft(n)
    circ.extend(sv.build_iqft(n).gates)
    got, want = run_both(n, circ, v)
    assert float(np.max(np.abs(got - want))) <= bound(len(circ))
    assert float(np.max(np.abs(got - v))) <= bound(len(circ))


@pytest.mark.parametrize("basis", [0, 5, 1234567])
def test_qft_basis_closed_form(basis):
    n = 22
    st = sv.init_basis_state(sv.Layout(n), basis % (1 << n), device=DEV)
    circ = sv.build_qft(n)
    sv.run_circuit(st, circ, fusion=TOL)
    err = float(np.max(np.abs(st.to_numpy() - oracle.dft_bit_reversed(n, basis % (1 << n)))))
    assert err <= bound(len(circ)), err


@pytest.mark.parametrize("frac,seed", [(0.0, 1), (0.5, 2), (1.0, 3)])
def test_random_circuits_tolerance(frac, seed):
    n = 18
    v = random_state(np.random.default_rng(seed), n)
    circ = sv.random_circuit(n, 300, np.random.default_rng(seed + 10), controlled_fraction=frac)
    got, want = run_both(n, circ, v)
    assert float(np.max(np.abs(got - want))) <= bound(len(circ))


def test_phase_heavy_stages_with_slot_and_outside_controls():
    """Diagonal gates of every flavour inside stage passes: controls on slot bits (register
    updates), outside the slots (folds), uncontrolled diagonals with q11 != 1 (F0 factors),
    and non-diagonal gates that force a flush in the middle of a stage."""
    n = 16
    rng = np.random.default_rng(77)
    ops = []
    for _ in range(12):
        t = int(rng.integers(8, 12))
        ops.append(sv.GateOp(sv.random_unitary(rng), t))
        for _ in range(10):
            c = int(rng.integers(0, n))
            if c == t:
                continue
            ph = np.exp(1j * rng.uniform(0, 2 * np.pi))
            d0 = 1.0 if rng.random() < 0.6 else np.exp(1j * rng.uniform(0, 2 * np.pi))
            ops.append(sv.GateOp(sv.GateMatrix(np.diag([d0, ph])), t, None if rng.random() < 0.2 else c))
    circ = sv.Circuit(n, ops)
    v = random_state(rng, n)
    got, want = run_both(n, circ, v)
    assert float(np.max(np.abs(got - want))) <= bound(len(circ))


def test_tolerance_passes_on_basis_zero_state():
    """Zeros everywhere (no speculation, no replay in this mode): still within the bound."""
    n = 16
    circ = sv.build_qft(n)
    st = sv.init_basis_state(sv.Layout(n), 0, device=DEV)
    sv.run_circuit(st, circ, fusion=TOL)
    assert float(np.max(np.abs(st.to_numpy() - oracle.dft_bit_reversed(n, 0)))) <= bound(len(circ))


@pytest.mark.parametrize("p", [1, 2])
def test_tolerance_passes_sharded_inproc(p):
    """Ranks in one process (global stages through k_exchange_stage, local passes in the mode)."""
    n = 16
    m = n - p
    v = random_state(np.random.default_rng(40 + p), n)
    circ = sv.build_qft(n)
    circ.extend(sv.random_circuit(n, 60, np.random.default_rng(p), controlled_fraction=0.4).gates)
    sts = [sv.LocalState(sv.Layout(n, p, r), torch.from_numpy(v[r << m:(r + 1) << m].copy()).to(DEV))
           for r in range(1 << p)]
    sv.run_circuit_inproc(sts, circ, sv.InprocFabric.group(sts), fusion=sv.FusionConfig(l_c=11, passes=True,
                                                                                          exact=False))
    torch.cuda.synchronize()
    got = np.concatenate([s.to_numpy() for s in sts])
    want = v.copy()
    oracle.run_circuit(want, circ.gates, threads=8)
    assert float(np.max(np.abs(got - want))) <= bound(len(circ))


def test_qft28_tolerance_full_size_vs_oracle():
    """Config-5 shape at n = 28: tolerance passes vs the oracle on the same state."""
    n = 28
    torch.cuda.empty_cache()
    st = sv.init_random_state(sv.Layout(n), seed=9, device=DEV)
    host = st.amps.cpu().numpy()
    circ = sv.build_qft(n)
    sv.run_circuit(st, circ, fusion=TOL)
    oracle.run_circuit(host, circ.gates, threads=16)
    want = torch.from_numpy(host).to(DEV)
    err = sv.max_abs_diff(st.amps, want)
    assert err <= bound(len(circ)), err
    del st, want, host
    torch.cuda.empty_cache()


def test_two_phase_stage_groups_mixed_diagonals():
    """k_dstage2 (eight targets per pass): runs on targets 6..9 then 10..13 with diagonal gates
    controlled by the other phase's targets (folds that must be flushed at the transpose),
    by slot bits (register updates), by low and high bits, uncontrolled diagonals with
    d0 != 1, non-diagonal gates in between (flushes), and controlled Hadamards."""
    n = 18
    rng = np.random.default_rng(123)
    ops = []
    for phase in ((6, 7, 8, 9), (10, 11, 12, 13)):
        for t in phase:
            ops.append(sv.GateOp(sv.hadamard(), t))
            for _ in range(9):
                c = int(rng.integers(0, n))
                if c == t:
                    continue
                ph = np.exp(1j * rng.uniform(0, 2 * np.pi))
                d0 = 1.0 if rng.random() < 0.7 else np.exp(1j * rng.uniform(0, 2 * np.pi))
                ops.append(sv.GateOp(sv.GateMatrix(np.diag([d0, ph])), t, None if rng.random() < 0.15 else c))
            if rng.random() < 0.5:
                c = int(rng.integers(0, n))
                ops.append(sv.GateOp(sv.random_unitary(rng), t, None if c == t else c))
    circ = sv.Circuit(n, ops)
    kinds = [p.kind for p in sv.plan_passes(circ.gates, n, 12, exact=False)]
    assert "local_stage2" in kinds, kinds
    v = random_state(rng, n)
    got, want = run_both(n, circ, v)
    assert float(np.max(np.abs(got - want))) <= bound(len(circ))


@pytest.mark.parametrize("n,l_c,seed", [(14, 12, 21), (16, 11, 22), (17, 12, 23), (19, 12, 24), (20, 10, 25)])
def test_scheduled_mixed_circuits_tolerance(n, l_c, seed):
    """Merged and reordered gates (passes.schedule_gates) through the tolerance kernels: Haar gates,
    Hadamards, (controlled) phase rotations and general diagonals on random placements -- the
    commutation-aware order must leave the state within the bound of the original order's."""
    rng = np.random.default_rng(seed)
    ops = []
    for _ in range(260):
        t = int(rng.integers(n))
        c = int((t + 1 + rng.integers(n - 1)) % n)
        kind = rng.random()
        if kind < 0.3:
            ops.append(sv.GateOp(sv.random_unitary(rng), t))
        elif kind < 0.5:
            ops.append(sv.GateOp(sv.random_unitary(rng), t, c))
        elif kind < 0.6:
            ops.append(sv.GateOp(sv.hadamard(), t))
        elif kind < 0.8:
            ops.append(sv.GateOp(sv.phase_r(int(rng.integers(2, 9))), t, c))
        elif kind < 0.9:
            ops.append(sv.GateOp(sv.phase_r(int(rng.integers(2, 9))), t))
        else:
            d = sv.GateMatrix.unchecked(np.diag(np.exp(1j * rng.uniform(0, 2 * np.pi, 2))))
            ops.append(sv.GateOp(d, t, c if rng.random() < 0.5 else None))
    circ = sv.Circuit(n, ops)
    fc = sv.FusionConfig(l_c=l_c, passes=True, exact=False)
    exact_plan = sv.plan_passes(circ.gates, n, sv.passes.tile_for(l_c, n))
    tol_plan = sv.plan_passes(circ.gates, n, sv.passes.tile_for(l_c, n), exact=False)
    assert len(tol_plan) <= len(exact_plan)
    v = random_state(rng, n)
    got, want = run_both(n, circ, v, fusion=fc)
    assert float(np.max(np.abs(got - want))) <= bound(len(circ))
