"""Pass planner host logic (CPU): grouping, rank-control resolution, rank-uniformity."""

from __future__ import annotations

import numpy as np

import paper_1601_07195_b200 as sv
from paper_1601_07195_b200.passes import _resolve_rank_controls, tile_for


def test_qft_plan_is_one_pass_per_four_stages():
    n, m = 30, 30
    circ = sv.build_qft(n)
    plan = sv.plan_passes(circ.gates, m, 12)
    # four consecutive transform stages H(k), R(k, c) for all c < k share one stage pass; the
    # last six (targets 0..5: a strided stage plus a leftover pass otherwise) are one low-bit pass
    # (k_dlow<exact>: one warp per 256 amplitudes)
    assert sv._lib.SV_MSTAGE_MAX_TARGETS == 4
    assert [p.kind for p in plan] == ["local_stage"] * 6 + ["local_low"]
    assert [sorted({op.target for op in p.gates}) for p in plan] == (
        [[k - 3, k - 2, k - 1, k] for k in range(29, 6, -4)] + [list(range(6))])
    assert [op for p in plan for op in p.gates] == list(circ.gates)
    assert max(len(p.gates) for p in plan) <= sv._lib.SV_MSTAGE_MAX_GATES


def test_random_circuit_plan_fuses_high_targets():
    """Tiles gather up to SV_TILE_GATHER high qubits: random circuits fuse several gates per pass."""
    circ = sv.random_circuit(30, 400, np.random.default_rng(1), controlled_fraction=0.3)
    plan = sv.plan_passes(circ.gates, 30, 12)
    assert [op for p in plan for op in p.gates] == list(circ.gates)
    assert len(circ) / len(plan) > 6.0
    G = sv._lib.SV_TILE_GATHER
    for p in plan:
        if p.kind == "local_tile":
            high = {op.target for op in p.gates if op.target >= 12 - G}
            assert len(high) <= G
        if p.kind == "local_stage":
            assert len({op.target for op in p.gates}) <= sv._lib.SV_MSTAGE_MAX_TARGETS


def test_global_stages_and_order_preserved():
    n, m = 12, 10
    circ = sv.build_qft(n)
    plan = sv.plan_passes(circ.gates, m, 0)
    assert [op for p in plan for op in p.gates] == list(circ.gates)
    glob = [p for p in plan if not p.local]
    assert [p.kind for p in glob] == ["global_stage", "global_stage"] and [p.target for p in glob] == [11, 10]
    assert all(len(p.gates) <= sv._lib.SV_STAGE_MAX_GATES for p in plan)


def test_plan_is_rank_independent_and_tile_bounds():
    rng = np.random.default_rng(3)
    circ = sv.random_circuit(16, 300, rng, controlled_fraction=0.5)
    for m in (13, 14, 16):
        a = sv.plan_passes(circ.gates, m, tile_for(12, m))
        b = sv.plan_passes(list(circ.gates), m, tile_for(12, m))
        assert a == b
        for p in a:
            if p.kind == "local_tile":  # low bits < T-G plus at most G gathered high bits
                G = sv._lib.SV_TILE_GATHER
                assert len({op.target for op in p.gates if op.target >= tile_for(12, m) - G}) <= G
            if p.kind == "local_stage":
                assert len({op.target for op in p.gates}) <= sv._lib.SV_MSTAGE_MAX_TARGETS and len(p.gates) > 1
    assert tile_for(5, 30) == 0 and tile_for(20, 30) == 13 and tile_for(12, 11) == 11


from hypothesis import given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402


@given(st.integers(9, 34), st.integers(0, 2**31 - 1), st.sampled_from([0, 9, 12, 13]))
@settings(max_examples=60, deadline=None)
def test_native_planner_invariants(m, seed, tile):
    """sv_plan_gates (the planner sv_apply_gates runs): order-preserving cover, one launch per
    group, tile groups gather at most G bits above T-G, stages span at most four targets."""
    rng = np.random.default_rng(seed)
    T = tile if tile and tile <= min(m, 13) else min(m, 13)
    zoo = [sv.hadamard(), sv.phase_r(3), sv.pauli_z(), sv.random_unitary(rng)]
    ops = []
    for _ in range(int(rng.integers(1, 400))):
        t = int(rng.integers(m)) if rng.random() < 0.7 else int(rng.integers(min(m, 6)))
        c = None if rng.random() < 0.5 else int((t + 1 + rng.integers(m - 1)) % m)
        ops.append(sv.GateOp(zoo[int(rng.integers(4))], t, c))
    plan = sv.plan_passes(ops, m, T if tile else 0)
    assert [op for p in plan for op in p.gates] == ops
    for p in plan:
        targets = {op.target for op in p.gates}
        if p.kind == "local_tile":
            assert len(p.gates) <= sv._lib.SV_FUSED_MAX_GATES
            G = sv._lib.SV_TILE_GATHER
            assert len({t for t in targets if t >= T - G}) <= G
        elif p.kind == "local_stage":
            assert len(targets) <= sv._lib.SV_MSTAGE_MAX_TARGETS and 1 < len(p.gates) <= sv._lib.SV_MSTAGE_MAX_GATES
        elif p.kind == "local_low":  # every target in qubits 0..5: one k_dlow pass
            assert max(targets) < 6 and len(p.gates) >= 2
        else:
            assert p.kind == "local_gate"


def test_planner_abi_errors():
    import ctypes

    from paper_1601_07195_b200 import _lib

    L = _lib.load()
    g = sv.kernels.gate_array([sv.GateOp(sv.hadamard(), 3)])
    ends = (ctypes.c_int32 * 4)()
    kinds = (ctypes.c_int32 * 4)()
    assert L.sv_plan_gates(3, g, 1, 0, ends, kinds, 4) == _lib.SV_EINVAL   # target 3 not local at m=3
    assert L.sv_plan_gates(20, g, 1, 14, ends, kinds, 4) == _lib.SV_EINVAL  # tile out of range
    assert L.sv_plan_gates(20, g, 1, 0, ends, kinds, 4) == 1 and kinds[0] == _lib.SV_GROUP_GATES
    assert L.sv_apply_group(None, 20, 1, g, 1, 0, None) == _lib.SV_EINVAL


def test_rank_controls_resolve_per_rank():
    lay0, lay1 = sv.Layout(8, 1, 0), sv.Layout(8, 1, 1)
    ops = [sv.GateOp(sv.hadamard(), 2, 7), sv.GateOp(sv.hadamard(), 3, 1), sv.GateOp(sv.hadamard(), 4)]
    r0 = _resolve_rank_controls(ops, lay0)
    r1 = _resolve_rank_controls(ops, lay1)
    assert [(o.target, o.control) for o in r0] == [(3, 1), (4, None)]
    assert [(o.target, o.control) for o in r1] == [(2, None), (3, 1), (4, None)]


def test_fusion_config_passes_flag_keeps_reference_plans():
    circ = sv.random_circuit(10, 50, np.random.default_rng(1))
    ref = sv.plan_fusion(circ, sv.FusionConfig(l_c=5))
    assert not ref.passes and all(isinstance(s, (sv.FusedBlockRun, sv.PassThrough)) for s in ref.segments)
    p = sv.plan_fusion(circ, sv.FusionConfig(l_c=5, passes=True))
    assert p.passes and p.flatten() == list(circ.gates)


def test_transform_stage_groups_take_the_compiled_path():
    """sv_stage_shape (pure host): the exact planner's stage groups of build_qft
    (circuits.py:141-156) are recognised as transform stages in circuit order (k_mstage with
    compiled control flow); a group with a foreign gate, or with a stage's phases out of
    order, stays with the run-dispatched kernel."""
    from paper_1601_07195_b200 import _lib
    from paper_1601_07195_b200.kernels import gate_array

    def shape(m, gates):
        gates = list(gates)
        return _lib.load().sv_stage_shape(m, gate_array(gates), len(gates))

    for n in (18, 26, 30, 33):
        groups = [p for p in sv.plan_passes(sv.build_qft(n).gates, n, 12) if p.kind == "local_stage"]
        assert groups
        assert all(shape(n, p.gates) == _lib.SV_SHAPE_FORWARD for p in groups)
    n = 26
    gates = list([p for p in sv.plan_passes(sv.build_qft(n).gates, n, 12) if p.kind == "local_stage"][0].gates)
    rng = np.random.default_rng(0)
    foreign = gates[:5] + [sv.GateOp(sv.random_unitary(rng), gates[0].target)] + gates[5:]
    assert shape(n, foreign) == _lib.SV_SHAPE_INTERPRETED
    swapped = gates[:]
    swapped[1], swapped[2] = swapped[2], swapped[1]  # the in-slot phases of the first stage out of order
    assert shape(n, swapped) == _lib.SV_SHAPE_INTERPRETED
    dropped = [g for k, g in enumerate(gates) if k % 7 != 3]  # still stages in order
    assert shape(n, dropped) == _lib.SV_SHAPE_FORWARD
    # inverse transform: the compiled inverse shape, after a compiled low-bit pass on stages 0..5
    plan = sv.plan_passes(sv.build_qft(n).inverse().gates, n, 12)
    assert plan[0].kind == "local_low" and len(plan[0].gates) == 21
    inv = [p for p in plan if p.kind == "local_stage"]
    assert inv and all(shape(n, p.gates) == _lib.SV_SHAPE_INVERSE for p in inv)
    # a forward stage list reversed WITHOUT conjugating is still inverse-shaped (phases are phases)
    rev = list(reversed(gates))
    assert shape(n, rev) == _lib.SV_SHAPE_INVERSE
