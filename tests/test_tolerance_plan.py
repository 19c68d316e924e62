"""Tolerance-mode planning on the host (CPU): the gate merge is an exact rewrite up to
rounding (checked with the dense Kronecker oracle, pkg/src/svsim/oracle.py:27-83), the
config refuses the mode without the pass planner, and plans are rank-independent."""

from __future__ import annotations

import numpy as np
import pytest

import paper_1601_07195_b200 as sv
from oracle import oracle


def test_exact_false_requires_passes():
    with pytest.raises(ValueError):
        sv.FusionConfig(l_c=12, exact=False)
    assert not sv.FusionConfig(l_c=12, passes=True, exact=False).exact


def test_merge_gates_matches_dense_oracle():
    rng = np.random.default_rng(5)
    n = 5
    for trial in range(20):
        ops = []
        for _ in range(30):
            t = int(rng.integers(0, n))
            if rng.random() < 0.4:
                c = int(rng.integers(0, n - 1))
                c = c + (c >= t)
                ops.append(sv.GateOp(sv.random_unitary(rng), t, c))
            else:
                ops.append(sv.GateOp(sv.random_unitary(rng), t))
            if rng.random() < 0.3:  # repeat the same placement right away: must merge
                ops.append(sv.GateOp(sv.random_unitary(rng), ops[-1].target, ops[-1].control))
        merged = sv.passes.merge_gates(ops)
        assert len(merged) < len(ops)
        v = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
        a = oracle.dense_run(n, ops, v)
        b = oracle.dense_run(n, merged, v)
        assert np.max(np.abs(a - b)) < 1e-12


def test_merge_respects_blocking_gates():
    h = sv.hadamard()
    ops = [sv.GateOp(h, 0), sv.GateOp(sv.pauli_x(), 1, 0), sv.GateOp(h, 0)]  # CNOT reads qubit 0 in between
    assert len(sv.passes.merge_gates(ops)) == 3
    ops = [sv.GateOp(h, 0), sv.GateOp(sv.pauli_x(), 2, 1), sv.GateOp(h, 0)]  # disjoint: H H merges
    assert len(sv.passes.merge_gates(ops)) == 2
    ops = [sv.GateOp(h, 0, 1), sv.GateOp(h, 1, 0)]  # same qubits, different roles: no merge
    assert len(sv.passes.merge_gates(ops)) == 2


def test_tolerance_plan_is_order_preserving_cover():
    circ = sv.build_qft(30)
    plan = sv.plan_passes(circ.gates, 30, 12, exact=False)
    flat = [op for p in plan for op in p.gates]
    assert len(flat) == len(circ)  # QFT has nothing to merge
    assert all(not p.exact for p in plan)
    # eight transform stages per two-phase pass, the last six stages (qubits 5..0) one low-bit pass
    assert [p.kind for p in plan] == ["local_stage2"] * 3 + ["local_low"]
    # the exact planner needs seven passes for the same circuit
    assert len(sv.plan_passes(circ.gates, 30, 12)) == 7


def _mixed_circuit(rng, n, count):
    """Haar gates, controlled Haar gates and (controlled) phase rotations on random placements."""
    ops = []
    for _ in range(count):
        t = int(rng.integers(0, n))
        c = int(rng.integers(0, n - 1))
        c = c + (c >= t)
        kind = rng.random()
        if kind < 0.35:
            ops.append(sv.GateOp(sv.random_unitary(rng), t))
        elif kind < 0.6:
            ops.append(sv.GateOp(sv.random_unitary(rng), t, c))
        elif kind < 0.85:
            ops.append(sv.GateOp(sv.phase_r(int(rng.integers(2, 7))), t, c))
        else:
            ops.append(sv.GateOp(sv.phase_r(int(rng.integers(2, 7))), t))
    return ops


def test_schedule_gates_is_a_commuting_reorder():
    """schedule_gates only moves gates past gates they commute with: same multiset of gates, and
    the same state as the original order on the dense oracle (kernels.py:120-131 semantics)."""
    rng = np.random.default_rng(11)
    n = 7
    moved = 0
    for trial in range(25):
        ops = _mixed_circuit(rng, n, 50)
        out = sv.passes.schedule_gates(ops, tile=5, gather=3)
        assert sorted(map(id, out)) == sorted(map(id, ops))
        moved += any(a is not b for a, b in zip(ops, out))
        v = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
        a = oracle.dense_run(n, ops, v)
        b = oracle.dense_run(n, out, v)
        assert np.max(np.abs(a - b)) < 1e-12
    assert moved > 20


def test_schedule_gates_keeps_non_commuting_order():
    h, x = sv.hadamard(), sv.pauli_x()
    # H(9) ; CNOT(9 -> 1) ; H(1): a chain through shared qubits, nothing may move
    ops = [sv.GateOp(h, 9), sv.GateOp(x, 1, 9), sv.GateOp(h, 1)]
    assert sv.passes.schedule_gates(ops, tile=5, gather=1) == ops
    # two controlled phases and a control share qubit 9 diagonally: free to reorder, all kept
    r = sv.phase_r(3)
    ops = [sv.GateOp(r, 9, 2), sv.GateOp(x, 3, 9), sv.GateOp(r, 9, 4)]
    assert len(sv.passes.schedule_gates(ops, tile=5, gather=1)) == 3


def test_tolerance_plan_packs_random_gates_into_fewer_passes():
    """Config-4 shape (25 Haar gates on uniform targets, n = 30): merged and reordered, the
    tolerance plan needs no more passes than the exact one and strictly fewer on most seeds;
    every rank-independent input gives the same plan twice."""
    fewer = 0
    for seed in range(8):
        circ = sv.random_circuit(30, 25, np.random.default_rng(seed), controlled_fraction=0.0)
        exact = sv.plan_passes(circ.gates, 30, 12)
        tol = sv.plan_passes(circ.gates, 30, 12, exact=False)
        assert len(tol) <= len(exact)
        fewer += len(tol) < len(exact)
        again = sv.plan_passes(circ.gates, 30, 12, exact=False)
        assert [(p.kind, len(p.gates)) for p in tol] == [(p.kind, len(p.gates)) for p in again]
    assert fewer >= 4


def _shape(m, gates):
    from paper_1601_07195_b200 import _lib
    from paper_1601_07195_b200.kernels import gate_array

    gates = list(gates)
    return _lib.load().sv_stage2_shape(m, gate_array(gates), len(gates))


def test_two_phase_groups_of_transforms_compile():
    """The two-phase groups of build_qft (circuits.py:141-156) run as compiled forward transform
    phases, those of its inverse as compiled inverse phases; any other two-phase group stays with
    the interpreter (sv_stage2_shape: pure host code)."""
    from paper_1601_07195_b200 import _lib

    for n in (18, 24, 30, 33):
        fwd = [p for p in sv.plan_passes(sv.build_qft(n).gates, n, 12, exact=False) if p.kind == "local_stage2"]
        inv = [p for p in sv.plan_passes(sv.build_qft(n).inverse().gates, n, 12, exact=False)
               if p.kind == "local_stage2"]
        assert fwd and inv
        assert all(_shape(n, p.gates) == _lib.SV_SHAPE_FORWARD for p in fwd)
        assert all(_shape(n, p.gates) == _lib.SV_SHAPE_INVERSE for p in inv)
    n = 24
    p = [p for p in sv.plan_passes(sv.build_qft(n).gates, n, 12, exact=False) if p.kind == "local_stage2"][0]
    gates = list(p.gates)
    # a general gate in place of a butterfly: not a transform shape any more
    k = next(i for i, g in enumerate(gates) if g.control is None)
    broken = gates[:k] + [sv.GateOp(sv.random_unitary(np.random.default_rng(0)), gates[k].target)] + gates[k + 1:]
    assert _shape(n, broken) == _lib.SV_SHAPE_INTERPRETED
    # a diagonal gate that is not a pure phase (d0 != 1)
    k = next(i for i, g in enumerate(gates) if g.control is not None)
    d = sv.GateMatrix.unchecked(np.diag([np.exp(0.3j), np.exp(0.7j)]))
    broken = gates[:k] + [sv.GateOp(d, gates[k].target, gates[k].control)] + gates[k + 1:]
    assert _shape(n, broken) == _lib.SV_SHAPE_INTERPRETED
    # not a two-phase group at all: an error, not a shape
    assert _shape(n, gates[:3]) < 0


def test_inverse_transform_plan_mirrors_the_forward_one():
    """Tolerance planner: the inverse of build_qft starts with the low-bit pass on stages 0..5 (not a
    78-gate tile of twelve stages) and continues with two-phase passes of eight stages; forward
    plans keep bits 0..3 out of two-phase groups (they end with a low-bit pass)."""
    for n in (20, 28, 30):
        fwd = sv.plan_passes(sv.build_qft(n).gates, n, 12, exact=False)
        inv = sv.plan_passes(sv.build_qft(n).inverse().gates, n, 12, exact=False)
        assert fwd[-1].kind == "local_low" and inv[0].kind == "local_low"
        assert len(inv[0].gates) == 21 and {op.target for op in inv[0].gates} == set(range(6))
        assert all(p.kind in ("local_stage2", "local_stage") for p in inv[1:])
        assert len(inv) <= len(fwd) + 1
        for p in fwd:
            if p.kind == "local_stage2":
                assert min(op.target for op in p.gates) >= 4
    # the cost model behind the choices is monotone in the obvious way
    from paper_1601_07195_b200.passes import plan_cost

    assert plan_cost(sv.plan_passes(sv.build_qft(30).gates, 30, 12, exact=False)) < 35.0
