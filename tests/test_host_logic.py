"""Host-side logic on CPU: register layout, gate matrices, per-rank routing, exchange plans,
fusion planning and traffic accounting -- the reference's contracts, no GPU needed."""

from __future__ import annotations

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_1601_07195_b200 as sv


def expected_exchange_counts(op, m, rank):
    """Per-rank (sent, received) bytes for one gate (restates pkg/tests/test_acceptance.py:61-71)."""
    case = sv.classify_case(op.target, op.control, m)
    if case is sv.BoundCase.SINGLE_REMOTE:
        return (1 << (m + 4), 1 << (m + 4))
    if case is sv.BoundCase.CONTROLLED_REMOTE_TARGET:
        return (1 << (m + 3), 1 << (m + 3))
    if case is sv.BoundCase.CONTROLLED_REMOTE_BOTH and (rank >> (op.control - m)) & 1:
        return (1 << (m + 4), 1 << (m + 4))
    return (0, 0)


class TestLayout:
    def test_index_round_trip(self):
        lay = sv.Layout(10, 3, 5)
        assert lay.m == 7 and lay.num_ranks == 8 and lay.local_len == 128
        for j in (0, 1, 77, 127):
            assert lay.split_global(lay.global_index(j)) == (5, j)

    def test_validation(self):
        with pytest.raises(ValueError):
            sv.Layout(0)
        with pytest.raises(sv.LayoutError):
            sv.Layout(4, 4)
        with pytest.raises(sv.LayoutError):
            sv.Layout(4, 1, 2)

    @given(st.integers(1, 40), st.data())
    @settings(max_examples=50, deadline=None)
    def test_global_split_property(self, n, data):
        p = data.draw(st.integers(0, n - 1))
        rank = data.draw(st.integers(0, (1 << p) - 1))
        lay = sv.Layout(n, p, rank)
        j = data.draw(st.integers(0, lay.local_len - 1))
        assert lay.split_global(lay.global_index(j)) == (rank, j)


class TestGateMatrix:
    def test_rejects_non_unitary(self):
        with pytest.raises(ValueError):
            sv.GateMatrix(np.array([[1, 0], [0, 2]], dtype=complex))

    def test_unchecked_and_dagger(self, rng):
        assert sv.GateMatrix.unchecked([[1, 0], [0, 2]]).mat[1, 1] == 2
        q = sv.random_unitary(rng)
        assert np.allclose(q.mat @ q.dagger().mat, np.eye(2), atol=1e-13)

    def test_abi_packing_order(self):
        q = sv.GateMatrix.unchecked([[1 + 2j, 3 + 4j], [5 + 6j, 7 + 8j]])
        assert list(q.qbuf()) == [1, 2, 3, 4, 5, 6, 7, 8]

    def test_read_only(self):
        with pytest.raises(ValueError):
            sv.hadamard().mat[0, 0] = 2


class TestPlanGate:
    @pytest.mark.parametrize("n,p", [(8, 1), (8, 2), (9, 3), (12, 3)])
    def test_traffic_matches_reference_accounting(self, n, p):
        m = n - p
        circ = sv.random_circuit(n, 300, np.random.default_rng(n * 10 + p))
        for op in circ:
            for rank in range(1 << p):
                a = sv.plan_gate(sv.Layout(n, p, rank), op.target, op.control)
                assert (a.sent, a.received) == expected_exchange_counts(op, m, rank)
                assert a.case is sv.classify_case(op.target, op.control, m)

    def test_partner_symmetry_and_half_coverage(self):
        n, p = 8, 3
        m = n - p
        for k in range(m, n):
            for rank in range(1 << p):
                a = sv.plan_gate(sv.Layout(n, p, rank), k, None)
                b = sv.plan_gate(sv.Layout(n, p, a.partner), k, None)
                assert b.partner == rank and a.own_is_zero != b.own_is_zero
                plan = sv.make_exchange_plan(sv.Layout(n, p, rank), k)
                assert plan.partner == a.partner
                assert (plan.this_rank_computes is sv.ComputesHalf.FIRST_HALF) == a.own_is_zero

    def test_case_routing(self):
        n, p = 8, 2
        m = n - p
        kinds = {}
        for rank in range(4):
            lay = sv.Layout(n, p, rank)
            kinds[rank] = (sv.plan_gate(lay, 1, 7).kind,        # case 4
                           sv.plan_gate(lay, 6, 7).kind,        # case 6
                           sv.plan_gate(lay, 7, 0).kind,        # case 5
                           sv.plan_gate(lay, 7, m - 1).c_local,
                           sv.plan_gate(lay, 0, 3).kind)        # case 3
        for rank, k in kinds.items():
            on = (rank >> 1) & 1
            assert k[0] == ("single" if on else "idle")
            assert k[1] == ("exchange" if on else "idle_exchange")
            assert k[2] == "exchange" and k[3] == m - 1 and k[4] == "controlled"

    def test_fence_classes_are_rank_uniform(self):
        """Every rank fences on exactly the same gates (collective calls must line up)."""
        n, p = 9, 3
        circ = sv.random_circuit(n, 200, np.random.default_rng(3))
        for op in circ:
            fenced = {sv.plan_gate(sv.Layout(n, p, r), op.target, op.control).fenced for r in range(8)}
            assert len(fenced) == 1


class TestExchangePlan:
    def test_default_chunk_is_saturation_floor(self):
        plan = sv.make_exchange_plan(sv.Layout(26, 1, 0), 25)
        assert plan.chunk_amps == sv.DEFAULT_CHUNK_BYTES // 16
        small = sv.make_exchange_plan(sv.Layout(8, 1, 0), 7)
        assert small.chunk_amps == small.half_amps and small.temp_capacity == small.chunk_amps

    def test_rejects_local_qubit(self):
        with pytest.raises(sv.LayoutError):
            sv.make_exchange_plan(sv.Layout(8, 1, 0), 3)
        with pytest.raises(sv.LayoutError):
            sv.make_exchange_plan(sv.Layout(8, 1, 0), 8)

    def test_plan_validation(self):
        good = dict(partner=1, this_rank_computes=sv.ComputesHalf.FIRST_HALF, chunk_amps=4, temp_capacity=8,
                    half_amps=8)
        sv.ExchangePlan(**good)
        for bad in ({"chunk_amps": 3}, {"temp_capacity": 4}, {"temp_capacity": 16}, {"chunk_amps": 0}):
            with pytest.raises(ValueError):
                sv.ExchangePlan(**{**good, **bad})


class TestFusionPlanning:
    def test_single_gate_is_one_run(self):
        plan = sv.plan_fusion(sv.Circuit(6, [sv.GateOp(sv.hadamard(), 0)]), sv.FusionConfig(l_c=5))
        assert len(plan.segments) == 1 and isinstance(plan.segments[0], sv.FusedBlockRun)

    def test_high_gate_splits_runs(self):
        circ = sv.Circuit(8, [sv.GateOp(sv.hadamard(), k) for k in (0, 7, 1)])
        kinds = [type(s) for s in sv.plan_fusion(circ, sv.FusionConfig(l_c=4)).segments]
        assert kinds == [sv.FusedBlockRun, sv.PassThrough, sv.FusedBlockRun]

    def test_disabled_and_flatten(self, rng):
        circ = sv.random_circuit(10, 60, rng)
        assert sv.plan_fusion(circ, sv.FusionConfig(l_c=5)).flatten() == list(circ.gates)
        off = sv.plan_fusion(circ, sv.FusionConfig(l_c=6, enabled=False))
        assert all(isinstance(s, sv.PassThrough) for s in off.segments)

    def test_iqft_leading_stages_form_one_run(self):
        n, l_c = 12, 8
        plan = sv.plan_fusion(sv.build_iqft(n), sv.FusionConfig(l_c=l_c))
        assert len(plan.segments[0].gates) == l_c * (l_c + 1) // 2

    def test_block_exponents(self):
        assert sv.default_block_exponent(32 << 20, m=30) == 20
        assert sv.default_block_exponent(32 << 20, m=10) == 10
        assert sv.gpu_block_exponent(30) == 13 and sv.gpu_block_exponent(9) == 9
        with pytest.raises(ValueError):
            sv.FusionConfig(l_c=0)


class TestPerfModel:
    def test_bound_table_m29(self):
        want = [0.43, 3.12, 0.21, 0.43, 1.56, 3.12]
        got = [sv.lower_bound_seconds(c, 29, sv.MachineParams()) for c in sv.BoundCase]
        assert max(abs(g - w) for g, w in zip(got, want)) <= 0.005

    def test_link_bytes_per_direction(self):
        assert sv.link_bytes_per_direction(sv.BoundCase.SINGLE_REMOTE, 33) == 1 << 37
        assert sv.link_bytes_per_direction(sv.BoundCase.CONTROLLED_REMOTE_TARGET, 33) == 1 << 36
        assert sv.link_bytes_per_direction(sv.BoundCase.SINGLE_LOCAL, 33) == 0

    def test_transform_gate_counts(self):
        assert [sv.build_qft(n).gate_count for n in (29, 34, 40)] == [435, 595, 820]
