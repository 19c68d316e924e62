"""GPU algebraic properties (the reference's hypothesis suite, pkg/tests/test_kernels.py:131-169,
run through the C ABI): norm preservation, U then U^dagger restores, involutions, disjoint
gates commute, fused == unfused -- on randomly drawn placements and states."""

from __future__ import annotations

import numpy as np
import pytest
import torch
from hypothesis import given, settings
from hypothesis import strategies as st

from conftest import random_state

pytestmark = pytest.mark.gpu

sv = pytest.importorskip("paper_1601_07195_b200")

DEV = "cuda:0"


def dev(v):
    return torch.from_numpy(np.ascontiguousarray(v)).to(DEV)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


@given(st.integers(0, 13), st.integers(0, 2**31 - 1))
@settings(max_examples=30, deadline=None)
def test_unitary_preserves_norm(k, seed):
    rng = np.random.default_rng(seed)
    n = 14
    a = dev(random_state(rng, n))
    sv.apply_single_raw(a, k, sv.random_unitary(rng))
    assert abs(float((a.abs() ** 2).sum().item()) - 1.0) < 1e-13


@given(st.integers(0, 2**31 - 1))
@settings(max_examples=25, deadline=None)
def test_gate_then_dagger_restores(seed):
    rng = np.random.default_rng(seed)
    n = 12
    v = random_state(rng, n)
    q = sv.random_unitary(rng)
    k = int(rng.integers(n))
    c = int(rng.integers(n))
    a = dev(v)
    if c == k:
        sv.apply_single_raw(a, k, q)
        sv.apply_single_raw(a, k, q.dagger())
    else:
        sv.apply_controlled_raw(a, c, k, q)
        sv.apply_controlled_raw(a, c, k, q.dagger())
    assert np.max(np.abs(host(a) - v)) < 1e-13


def test_involutions():
    rng = np.random.default_rng(1)
    v = random_state(rng, 10)
    for q in (sv.pauli_x(), sv.hadamard(), sv.pauli_y(), sv.pauli_z()):
        for k in (0, 4, 9):
            a = dev(v)
            sv.apply_single_raw(a, k, q)
            sv.apply_single_raw(a, k, q)
            assert np.max(np.abs(host(a) - v)) < 1e-13


@given(st.integers(0, 2**31 - 1))
@settings(max_examples=20, deadline=None)
def test_disjoint_gates_commute(seed):
    rng = np.random.default_rng(seed)
    n = 12
    v = random_state(rng, n)
    qs = rng.permutation(n)[:3]
    a_gate, b_gate = sv.random_unitary(rng), sv.random_unitary(rng)
    ab, ba = dev(v), dev(v)
    sv.apply_single_raw(ab, int(qs[0]), a_gate)
    sv.apply_controlled_raw(ab, int(qs[1]), int(qs[2]), b_gate)
    sv.apply_controlled_raw(ba, int(qs[1]), int(qs[2]), b_gate)
    sv.apply_single_raw(ba, int(qs[0]), a_gate)
    assert np.max(np.abs(host(ab) - host(ba))) < 1e-14


@given(st.integers(0, 2**31 - 1), st.sampled_from([9, 10, 12, 13]))
@settings(max_examples=15, deadline=None)
def test_fused_and_passes_bitwise_equal_unfused(seed, l_c):
    rng = np.random.default_rng(seed)
    n = 15
    v = random_state(rng, n)
    circ = sv.random_circuit(n, 60, rng, controlled_fraction=0.5)
    ref = sv.state_from_global(sv.Layout(n), v, device=DEV)
    sv.run_circuit(ref, circ)
    want = host(ref.amps)
    for fusion in (sv.FusionConfig(l_c=l_c), sv.FusionConfig(l_c=l_c, passes=True)):
        s = sv.state_from_global(sv.Layout(n), v, device=DEV)
        sv.run_circuit(s, circ, fusion=fusion)
        assert np.array_equal(host(s.amps).view(np.uint64), want.view(np.uint64)), fusion


def test_long_circuit_norm_n20():
    """Reference acceptance criterion: 1000 random gates at n=20 keep the norm within 1e-10."""
    for seed in (11, 12):
        circ = sv.random_circuit(20, 1000, np.random.default_rng(seed))
        s = sv.init_basis_state(sv.Layout(20), device=DEV)
        sv.run_circuit(s, circ, fusion=sv.FusionConfig(l_c=13, passes=True))
        assert abs(1.0 - sv.global_norm_sq(s)) <= 1e-10


@given(st.integers(9, 16), st.integers(0, 2**31 - 1), st.sampled_from([0, 9, 10, 12]),
       st.floats(0.0, 0.6), st.booleans())
@settings(max_examples=40, deadline=None)
def test_native_planner_bitwise_fuzz(n, seed, tile, zero_frac, structured):
    """sv_apply_gates on random gate lists (every update shape, controls anywhere, runs that
    favour stages or tiles, states salted with +-0) equals the oracle's unfused, unspecialised
    evaluation bit for bit -- tiles, multi-target stages, speculation and replays included."""
    from oracle import oracle

    rng = np.random.default_rng(seed)
    v = random_state(rng, n)
    if zero_frac:
        f = v.view(np.float64)
        hit = rng.random(f.shape) < zero_frac
        f[hit] = np.where(rng.random(hit.sum()) < 0.5, 0.0, -0.0)
    th = float(rng.uniform(0, 2 * np.pi))
    zoo = [sv.random_unitary(rng), sv.hadamard(), sv.phase_r(int(rng.integers(1, 9))), sv.pauli_z(),
           sv.pauli_x(), sv.rotation_y(th), sv.rotation_z(th), sv.GateMatrix.unchecked([[1, 0], [0, 0.5 + 0.5j]]),
           sv.GateMatrix.unchecked([[0.5, 0.5], [0.5, -0.5]])]
    hot = [int(x) for x in rng.choice(n, 3, replace=False)]
    ops = []
    for _ in range(int(rng.integers(1, 160))):
        t = hot[int(rng.integers(3))] if structured and rng.random() < 0.8 else int(rng.integers(n))
        c = None if rng.random() < 0.4 else int((t + 1 + rng.integers(n - 1)) % n)
        ops.append(sv.GateOp(zoo[int(rng.integers(len(zoo)))], t, c))
    T = tile if tile and tile <= min(n, 13) else 0
    a = dev(v)
    sv.kernels.apply_gates(a, ops, tile=T)
    w = v.copy()
    oracle.run_circuit(w, ops, threads=4)
    assert np.array_equal(host(a).view(np.uint64), w.view(np.uint64))
