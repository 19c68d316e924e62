"""Pass planner host logic (CPU): grouping, rank-control resolution, rank-uniformity."""

from __future__ import annotations

import numpy as np

import paper_1601_07195_b200 as sv
from paper_1601_07195_b200.passes import _resolve_rank_controls, tile_for


def test_qft_plan_is_one_pass_per_high_stage():
    n, m = 30, 30
    circ = sv.build_qft(n)
    plan = sv.plan_passes(circ.gates, m, 12)
    kinds = [p.kind for p in plan]
    # every high transform stage is one same-target pass, the low stages one register-tiled run
    k = kinds.index("local_tile")
    assert kinds[:k] == ["local_stage"] * k and kinds[k:] == ["local_tile"] and 18 <= k <= 24
    assert [p.target for p in plan[:k]] == list(range(29, 29 - k, -1))
    assert [op for p in plan for op in p.gates] == list(circ.gates)


def test_random_circuit_plan_fuses_high_targets():
    """Tiles gather up to four high qubits: random circuits fuse several gates per pass."""
    circ = sv.random_circuit(30, 400, np.random.default_rng(1), controlled_fraction=0.3)
    plan = sv.plan_passes(circ.gates, 30, 12)
    assert [op for p in plan for op in p.gates] == list(circ.gates)
    assert len(circ) / len(plan) > 4.0
    for p in plan:
        if p.kind == "local_tile":
            high = {op.target for op in p.gates if op.target >= 8}
            assert len(high) <= 4
        if p.kind == "local_stage":
            assert len({op.target for op in p.gates}) == 1


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
            if p.kind == "local_tile":  # low bits < T-4 plus at most four gathered high bits
                assert len({op.target for op in p.gates if op.target >= tile_for(12, m) - 4}) <= 4
            if p.kind == "local_stage":
                assert len({op.target for op in p.gates}) == 1 and p.target >= 5
    assert tile_for(5, 30) == 0 and tile_for(20, 30) == 13 and tile_for(12, 11) == 11


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
