"""GPU: multi-target stage passes (k_mstage) -- bitwise against the oracle.

One stage launch applies a run of gates whose targets lie in at most four
qubits; controls anywhere: on a slot bit (compile-time pair pattern), on a lane
bit (per-lane), above the lanes (warp-uniform ballot), including runs longer
than 32 gates (several ballot chunks) and the 128-gate maximum.  Every update
shape (general, real, Hadamard-like, diagonal, phase) is in the zoo, and
zero-salted states force the exact replay.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import random_state
from test_gpu_passes import DEV, bits_equal, gate_zoo, run_oracle, with_zeros

pytestmark = pytest.mark.gpu

sv = pytest.importorskip("paper_1601_07195_b200")
from paper_1601_07195_b200 import _lib  # noqa: E402
from paper_1601_07195_b200.kernels import device_view, gate_array, stream_handle  # noqa: E402


def apply_stage(a, ops):
    ptr, m = device_view(a)
    rc = _lib.load().sv_apply_group(ptr, m, _lib.SV_GROUP_STAGE, gate_array(ops), len(ops), 0, stream_handle())
    _lib.check(rc)


def stage_ops(rng, n, targets, count, cfrac=0.7, controls=None):
    zoo = gate_zoo(rng) + [sv.GateMatrix.unchecked([[0.5, -0.25], [0.75, 1.5]]),  # real, not unitary
                           sv.GateMatrix.unchecked([[0.25, 0.25], [0.25, -0.25]])]  # Hadamard-like
    ops = []
    for _ in range(count):
        t = int(targets[int(rng.integers(len(targets)))])
        c = None
        if rng.random() < cfrac:
            pool = controls if controls is not None else range(n)
            cands = [x for x in pool if x != t]
            c = int(cands[int(rng.integers(len(cands)))])
        ops.append(sv.GateOp(zoo[int(rng.integers(len(zoo)))], t, c))
    return ops


@pytest.mark.parametrize("n,targets", [(8, [5, 6, 7]), (12, [11, 3, 7]), (14, [0, 1, 2]), (16, [9]),
                                       (16, [15, 4]), (18, [17, 16, 15]), (20, [8, 0, 19]), (10, [6, 7, 8, 9]),
                                       (16, [0, 1, 2, 3]), (20, [19, 3, 11, 0]), (22, [21, 20, 19, 18])])
def test_stage_runs_bitwise(n, targets):
    rng = np.random.default_rng(4000 + 31 * n + sum(targets))
    for trial in range(3):
        v = with_zeros(rng, n) if trial == 2 else random_state(rng, n)
        ops = stage_ops(rng, n, targets, [20, 77, 128][trial])
        a = torch.from_numpy(v.copy()).to(DEV)
        apply_stage(a, ops)
        torch.cuda.synchronize()
        assert bits_equal(a.cpu().numpy(), run_oracle(v, ops)), (n, targets, trial)


@pytest.mark.parametrize("nslots", [3, 4])
@pytest.mark.parametrize("ctl", ["lanes", "warp", "cta", "slots"])
def test_stage_control_placements(ctl, nslots):
    """Controls only on lane bits (0..4), warp bits (5..7), CTA bits (above the slots) or the slot bits."""
    n, targets = 17 + nslots - 3, list(range(8, 8 + nslots))
    pool = {"lanes": range(5), "warp": range(5, 8), "cta": range(8 + nslots, n), "slots": targets}[ctl]
    rng = np.random.default_rng({"lanes": 1, "warp": 2, "cta": 3, "slots": 4}[ctl] + 10 * nslots)
    v = random_state(rng, n)
    ops = stage_ops(rng, n, targets, 100, cfrac=0.9, controls=list(pool))
    a = torch.from_numpy(v.copy()).to(DEV)
    apply_stage(a, ops)
    torch.cuda.synchronize()
    assert bits_equal(a.cpu().numpy(), run_oracle(v, ops)), ctl


def test_stage_replay_on_zero_results():
    """Basis states (mostly exact zeros) and mid-chain cancellations take the exact replay."""
    n = 15
    rng = np.random.default_rng(7)
    for v in (np.eye(1, 1 << n, 1234, dtype=np.complex128)[0], np.full(1 << n, 0.5 + 0.5j)):
        ops = [sv.GateOp(sv.hadamard(), 14)]
        ops += [sv.GateOp(sv.GateMatrix.unchecked([[1, 0], [0, 0.5 + 0.5j]]), t, c)
                for t, c in zip([14, 13, 12] * 10, rng.integers(0, 12, 30))]
        ops += stage_ops(rng, n, [12, 13, 14], 40)
        a = torch.from_numpy(v.copy()).to(DEV)
        apply_stage(a, ops)
        torch.cuda.synchronize()
        assert bits_equal(a.cpu().numpy(), run_oracle(v, ops))


def test_qft_plan_runs_through_stages_bitwise():
    n = 21
    rng = np.random.default_rng(21)
    v = with_zeros(rng, n, frac=0.05)
    circ = sv.build_qft(n)
    st = sv.LocalState(sv.Layout(n), torch.from_numpy(v.copy()).to(DEV))
    sv.run_circuit(st, circ, fusion=sv.FusionConfig(l_c=12, passes=True))
    torch.cuda.synchronize()
    assert bits_equal(st.amps.cpu().numpy(), run_oracle(v, circ.gates))


def test_stage_abi_guards():
    a = torch.zeros(1 << 10, dtype=torch.complex128, device=DEV)
    ptr, m = device_view(a)
    L = _lib.load()
    five = [sv.GateOp(sv.hadamard(), t) for t in (1, 2, 3, 4, 5)]
    assert L.sv_apply_group(ptr, m, _lib.SV_GROUP_STAGE, gate_array(five), 5, 0, stream_handle()) == _lib.SV_EINVAL
    assert "distinct targets" in L.sv_last_error().decode()
    small = torch.zeros(1 << 3, dtype=torch.complex128, device=DEV)  # fewer bits than slots
    sptr, sm = device_view(small)
    assert L.sv_apply_group(sptr, sm, _lib.SV_GROUP_STAGE, gate_array(five[:2]), 2, 0, stream_handle()) == _lib.SV_EINVAL
    many = [sv.GateOp(sv.hadamard(), 1)] * (_lib.SV_MSTAGE_MAX_GATES + 1)
    assert L.sv_apply_group(ptr, m, _lib.SV_GROUP_STAGE, gate_array(many), len(many), 0,
                            stream_handle()) == _lib.SV_EINVAL


@pytest.mark.parametrize("n", [4, 5, 6, 7, 8])
def test_stage_tiny_slices_partial_warps(n):
    """Slices with fewer than 32 groups (partial warps take part in the ballots with dummy rows)."""
    rng = np.random.default_rng(600 + n)
    for trial in range(4):
        v = with_zeros(rng, n) if trial % 2 else random_state(rng, n)
        targets = [int(t) for t in rng.choice(n, min(_lib.SV_MSTAGE_MAX_TARGETS, n), replace=False)]
        ops = stage_ops(rng, n, targets, [5, 40, 77, 128][trial])
        a = torch.from_numpy(v.copy()).to(DEV)
        apply_stage(a, ops)
        torch.cuda.synchronize()
        assert bits_equal(a.cpu().numpy(), run_oracle(v, ops)), (n, trial)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_stage_all_zero_groups_sign_replay(seed):
    """Groups whose 16 amplitudes are all +-0 replay on sign bits (ms_replay_zero): random zero
    signs in whole zero blocks, every gate kind, slot / warp / CTA / lane controls."""
    n = 16
    rng = np.random.default_rng(900 + seed)
    v = random_state(rng, n)
    idx = np.arange(1 << n)
    dead = ((idx >> 11) & 3) != 0  # three quarters of the state in whole zero blocks
    f = v.view(np.float64).reshape(-1, 2)
    f[dead] = np.where(rng.random((dead.sum(), 2)) < 0.5, 0.0, -0.0)
    for targets in ([7, 8, 9, 10], [0, 3, 5, 9], [2, 6]):
        ops = stage_ops(rng, n, targets, 100, cfrac=0.7)
        a = torch.from_numpy(v.copy()).to(DEV)
        apply_stage(a, ops)
        torch.cuda.synchronize()
        assert bits_equal(a.cpu().numpy(), run_oracle(v, ops)), targets
    basis = np.zeros(1 << n, dtype=np.complex128)
    basis[int(rng.integers(1 << n))] = 1.0
    ops = stage_ops(rng, n, [12, 13, 14, 15], 120)
    a = torch.from_numpy(basis.copy()).to(DEV)
    apply_stage(a, ops)
    torch.cuda.synchronize()
    assert bits_equal(a.cpu().numpy(), run_oracle(basis, ops))


# ---------------------------------------------------------------- exact low-bit groups (k_dlow<exact>)

def apply_low(a, ops):
    ptr, m = device_view(a)
    rc = _lib.load().sv_apply_group(ptr, m, _lib.SV_GROUP_LOW, gate_array(ops), len(ops), 0, stream_handle())
    _lib.check(rc)


@pytest.mark.parametrize("n", [11, 12, 15, 19])
def test_low_groups_bitwise(n):
    """Runs of gates with every target in qubits 0..5 as ONE exact low-bit pass: every update shape,
    controls on register bits, lane bits and bits above the block; dense, zero-salted and basis
    states (the latter two take the warp's exact replay).  Bitwise against the oracle."""
    rng = np.random.default_rng(9100 + n)
    for trial in range(4):
        ops = stage_ops(rng, n, list(range(6)), [7, 40, 96, 64][trial], cfrac=0.6)
        if trial == 2:
            v = with_zeros(rng, n)
        elif trial == 3:
            v = np.zeros(1 << n, dtype=np.complex128)
            v[int(rng.integers(1 << n))] = 1.0
        else:
            v = random_state(rng, n)
        a = torch.from_numpy(v.copy()).to(DEV)
        apply_low(a, ops)
        torch.cuda.synchronize()
        assert bits_equal(a.cpu().numpy(), run_oracle(v, ops)), (n, trial)


def test_low_group_is_the_transform_tail():
    """The exact planner gives the last six stages of build_qft to one low-bit pass, and the pass
    plan stays bit-identical to per-gate execution on dense and on basis inputs."""
    n = 18
    circ = sv.build_qft(n)
    plan = sv.plan_passes(circ.gates, n, 12)
    assert plan[-1].kind == "local_low" and {op.target for op in plan[-1].gates} == set(range(6))
    rng = np.random.default_rng(77)
    basis = np.zeros(1 << n, dtype=np.complex128)
    basis[12345] = 1.0
    for v in (random_state(rng, n), basis):
        st = sv.state_from_global(sv.Layout(n), v, device=DEV)
        sv.run_circuit(st, circ, fusion=sv.FusionConfig(l_c=12, passes=True))
        torch.cuda.synchronize()
        assert bits_equal(st.to_numpy(), run_oracle(v, list(circ.gates)))


def test_inverse_transform_exact_plan_bitwise():
    """The exact plan of the inverse transform mirrors the forward one -- a compiled low-bit pass on
    stages 0..5, then compiled inverse stage groups -- and stays bit-identical to per-gate execution
    on dense, zero-salted and basis inputs; sub-tails (stages 0..t0) too."""
    from paper_1601_07195_b200 import _lib

    n = 18
    circ = sv.build_qft(n).inverse()
    plan = sv.plan_passes(circ.gates, n, 12)
    assert plan[0].kind == "local_low" and len(plan[0].gates) == 21
    for p in plan[1:]:
        assert p.kind == "local_stage"
        assert _lib.load().sv_stage_shape(n, gate_array(list(p.gates)), len(p.gates)) == _lib.SV_SHAPE_INVERSE
    rng = np.random.default_rng(78)
    basis = np.zeros(1 << n, dtype=np.complex128)
    basis[54321] = 1.0
    for v in (random_state(rng, n), with_zeros(rng, n), basis):
        st = sv.state_from_global(sv.Layout(n), v, device=DEV)
        sv.run_circuit(st, circ, fusion=sv.FusionConfig(l_c=12, passes=True))
        torch.cuda.synchronize()
        assert bits_equal(st.to_numpy(), run_oracle(v, list(circ.gates)))
    for t0 in (1, 2, 3, 4, 5):  # inverse and forward sub-tails as single low-bit groups
        fwd = [op for op in sv.build_qft(n).gates if op.target <= t0]
        for ops in (fwd, [op.dagger() for op in reversed(fwd)]):
            if len(ops) < 2:
                continue
            for v in (random_state(rng, 13), with_zeros(rng, 13)):
                a = torch.from_numpy(v.copy()).to(DEV)
                apply_low(a, ops)
                torch.cuda.synchronize()
                assert bits_equal(a.cpu().numpy(), run_oracle(v, ops)), t0


def test_low_group_rejects_high_targets():
    a = torch.zeros(1 << 12, dtype=torch.complex128, device=DEV)
    with pytest.raises(Exception):
        apply_low(a, [sv.GateOp(sv.hadamard(), 7), sv.GateOp(sv.hadamard(), 1)])


# ------------------------------------------- compiled stage groups (k_mstage<true>) and their fallbacks

def _transform_stage_group(n, slots, rng, drop=0.0, shuffle_in_slot=False, extra=None):
    """H(t), R(t, c) for all c < t, for t in `slots` (descending): the stage group of build_qft
    (circuits.py:141-156) on arbitrary slot qubits, optionally with gates dropped at random."""
    ops = []
    for t in sorted(slots, reverse=True):
        block = [sv.GateOp(sv.hadamard(), t)]
        ctl = list(range(t - 1, -1, -1))
        if shuffle_in_slot:
            rng.shuffle(ctl)
        block += [sv.GateOp(sv.phase_r(t - c + 1), t, c) for c in ctl]
        ops += [g for g in block if rng.random() >= drop]
    if extra is not None:
        ops.insert(int(rng.integers(len(ops) + 1)), extra)
    return ops


@pytest.mark.parametrize("n,slots", [(14, [13, 12, 11, 10]), (16, [15, 14, 13, 12]), (18, [12, 11, 10, 9]),
                                     (15, [14, 9, 8, 3]), (20, [19, 18, 17]), (13, [12, 11]), (17, [8, 7, 6, 5])])
def test_compiled_stage_groups_bitwise(n, slots):
    """Transform-shaped stage groups take the compiled control flow (k_mstage<true>); with gates
    dropped, reordered or a foreign gate inserted they either still match or fall back to the
    dispatched kernel -- every variant bitwise equal to the oracle, on dense, zero-salted and
    basis states."""
    rng = np.random.default_rng(5200 + 17 * n + sum(slots))
    variants = [
        _transform_stage_group(n, slots, rng),
        _transform_stage_group(n, slots, rng, drop=0.3),
        _transform_stage_group(n, slots, rng, drop=0.6),
        _transform_stage_group(n, slots, rng, shuffle_in_slot=True),
        _transform_stage_group(n, slots, rng, extra=sv.GateOp(sv.random_unitary(rng), slots[0])),
        _transform_stage_group(n, slots, rng, extra=sv.GateOp(sv.phase_r(3), slots[-1], slots[0])),
    ]
    # the inverse stages (gates reversed and conjugated): the compiled inverse shape and its fallbacks
    variants += [[op.dagger() for op in reversed(v)] for v in variants[:5]]
    basis = np.zeros(1 << n, dtype=np.complex128)
    basis[int(rng.integers(1 << n))] = 1.0
    for vi, ops in enumerate(variants):
        ops = ops[:128]
        if len(ops) < 2:
            continue
        for v in (random_state(rng, n), with_zeros(rng, n), basis):
            a = torch.from_numpy(v.copy()).to(DEV)
            apply_stage(a, ops)
            torch.cuda.synchronize()
            assert bits_equal(a.cpu().numpy(), run_oracle(v, ops)), (n, slots, vi)
