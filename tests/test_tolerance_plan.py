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
