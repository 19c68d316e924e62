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
