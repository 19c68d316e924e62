"""GPU: register-tiled runs, same-target stages, structure-specialised updates and pass fusion.

Strictest bar: the raw bit patterns (sign of zero included) equal the oracle's
unfused, unspecialised evaluation of the reference arithmetic.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import random_state
from test_gpu_exchange import run_loopback

pytestmark = pytest.mark.gpu

sv = pytest.importorskip("paper_1601_07195_b200")
from oracle import oracle  # noqa: E402

DEV = "cuda:0"


def bits_equal(a, b):
    return np.array_equal(np.ascontiguousarray(a).view(np.uint64), np.ascontiguousarray(b).view(np.uint64))


def with_zeros(rng, n, frac=0.15):
    """Random state with some exact +-0 components (exercises the exact-zero branches)."""
    v = random_state(rng, n)
    f = v.view(np.float64).copy()
    hit = rng.random(f.shape) < frac
    f[hit] = np.where(rng.random(hit.sum()) < 0.5, 0.0, -0.0)
    return f.view(np.complex128)


def gate_zoo(rng):
    """General, diagonal, phase (incl. -0 imaginary parts), real and anti-diagonal matrices."""
    th = rng.uniform(0, 2 * np.pi)
    return [
        sv.random_unitary(rng), sv.hadamard(), sv.phase_r(int(rng.integers(1, 9))),
        sv.phase_r(int(rng.integers(1, 9))).dagger(), sv.rotation_z(th), sv.pauli_z(), sv.pauli_x(),
        sv.GateMatrix([[np.exp(1j * th), 0], [0, np.exp(-2j * th)]]), sv.pauli_y(), sv.rotation_y(th),
    ]


def random_ops(rng, n, count, tmax, cfrac=0.5, zoo=True):
    ops = []
    for _ in range(count):
        g = gate_zoo(rng)[int(rng.integers(10))] if zoo and rng.random() < 0.6 else sv.random_unitary(rng)
        t = int(rng.integers(tmax))
        c = None
        if rng.random() < cfrac:
            c = int(rng.integers(n - 1))
            c = c + 1 if c >= t else c
        ops.append(sv.GateOp(g, t, c))
    return ops


def run_oracle(v, ops):
    w = v.copy()
    oracle.run_circuit(w, ops, threads=8)
    return w


@pytest.mark.parametrize("n,T", [(9, 9), (12, 12), (13, 13), (16, 12), (16, 13), (18, 10)])
def test_tile_runs_bitwise(n, T):
    rng = np.random.default_rng(1000 + 17 * n + T)
    for trial in range(3):
        v = with_zeros(rng, n) if trial else random_state(rng, n)
        ops = random_ops(rng, n, 120, T)
        a = torch.from_numpy(v.copy()).to(DEV)
        sv.kernels.apply_gates(a, ops, tile=T)
        torch.cuda.synchronize()
        assert bits_equal(a.cpu().numpy(), run_oracle(v, ops)), (n, T, trial)


@pytest.mark.parametrize("T", [9, 10, 12, 13])
def test_gathered_tile_groups_bitwise(T):
    """Forced SV_GROUP_TILE groups whose targets are SV_TILE_GATHER high slice bits spread over
    the whole slice (top bit included) plus the contiguous low bits; controls on register,
    thread (warp and lane) and above-tile bits.  Bitwise vs the oracle."""
    from paper_1601_07195_b200 import _lib
    from paper_1601_07195_b200.kernels import device_view, gate_array, stream_handle

    n, G = 20, sv._lib.SV_TILE_GATHER
    rng = np.random.default_rng(77 + T)
    for trial in range(3):
        high = sorted(int(x) for x in rng.choice(np.arange(T - G, n), G, replace=False))
        if trial == 0:
            high[-1] = n - 1
        tset = list(range(T - G)) + high
        ops = []
        for _ in range(150):
            t = tset[int(rng.integers(len(tset)))]
            c = None if rng.random() < 0.4 else int(rng.integers(n - 1))
            c = None if c is None else (c + 1 if c >= t else c)
            g = gate_zoo(rng)[int(rng.integers(10))] if rng.random() < 0.5 else sv.random_unitary(rng)
            ops.append(sv.GateOp(g, t, c))
        v = with_zeros(rng, n) if trial else random_state(rng, n)
        a = torch.from_numpy(v.copy()).to(DEV)
        ptr, m = device_view(a)
        assert _lib.load().sv_apply_group(ptr, m, _lib.SV_GROUP_TILE, gate_array(ops), len(ops), T,
                                          stream_handle()) == 0, _lib.load().sv_last_error()
        torch.cuda.synchronize()
        assert bits_equal(a.cpu().numpy(), run_oracle(v, ops)), (T, trial, high)


def test_tile_group_rejects_too_many_gathered_bits():
    """A forced tile group with SV_TILE_GATHER + 1 distinct targets above the contiguous bits is
    refused (SV_EINVAL, state untouched), exactly G is accepted."""
    from paper_1601_07195_b200 import _lib
    from paper_1601_07195_b200.kernels import device_view, gate_array, stream_handle

    n, T, G = 20, 12, sv._lib.SV_TILE_GATHER
    v = random_state(np.random.default_rng(3), n)
    a = torch.from_numpy(v.copy()).to(DEV)
    ptr, m = device_view(a)
    L = _lib.load()
    too_many = [sv.GateOp(sv.hadamard(), t) for t in range(T - G, T - G + G + 1)]
    assert L.sv_apply_group(ptr, m, _lib.SV_GROUP_TILE, gate_array(too_many), len(too_many), T,
                            stream_handle()) == _lib.SV_EINVAL
    torch.cuda.synchronize()
    assert bits_equal(a.cpu().numpy(), v)
    ok = too_many[:G]
    assert L.sv_apply_group(ptr, m, _lib.SV_GROUP_TILE, gate_array(ok), len(ok), T, stream_handle()) == 0
    torch.cuda.synchronize()
    assert bits_equal(a.cpu().numpy(), run_oracle(v, ok))


def test_tile_register_set_transitions_and_natural_layout():
    """Target sequences that hit the natural layout, force many transposes, or repeat one target."""
    n = 14
    rng = np.random.default_rng(5)
    v = with_zeros(rng, n)
    for targets in ([12, 11, 10, 9] * 5, list(range(13)) * 3, [0] * 40, [3, 12, 0, 7, 12, 1, 9, 4, 11, 2, 5],
                    [12, 11, 10, 9, 0, 12]):
        ops = [sv.GateOp(sv.random_unitary(rng), t, None if i % 3 else (t + 5) % n) for i, t in enumerate(targets)]
        a = torch.from_numpy(v.copy()).to(DEV)
        sv.kernels.apply_gates(a, ops, tile=13)
        torch.cuda.synchronize()
        assert bits_equal(a.cpu().numpy(), run_oracle(v, ops)), targets


@pytest.mark.parametrize("n", [14, 20])
def test_stage_passes_and_mixed_lists_bitwise(n):
    rng = np.random.default_rng(n)
    v = with_zeros(rng, n)
    ops = []
    for k in (n - 1, 15, 13, 9, 4):  # stages on high and low targets, any controls
        k = min(k, n - 1)
        ops.append(sv.GateOp(sv.hadamard(), k))
        ops += [sv.GateOp(g, k, c) for c, g in zip(rng.permutation([c for c in range(n) if c != k])[:7],
                                                     gate_zoo(rng))]
    ops += random_ops(rng, n, 60, n)
    a = torch.from_numpy(v.copy()).to(DEV)
    sv.kernels.apply_gates(a, ops)
    torch.cuda.synchronize()
    assert bits_equal(a.cpu().numpy(), run_oracle(v, ops))


@pytest.mark.parametrize("n", [12, 16, 21])
def test_qft_iqft_pass_fusion_bitwise(n):
    rng = np.random.default_rng(70 + n)
    for build in (sv.build_qft, sv.build_iqft):
        circ = build(n)
        for v in (random_state(rng, n), np.eye(1, 1 << n, int(rng.integers(1 << n)), dtype=np.complex128)[0]):
            want = run_oracle(v, circ.gates)
            for l_c in (9, 12, 13):
                st = sv.state_from_global(sv.Layout(n), v, device=DEV)
                sv.run_circuit(st, circ, fusion=sv.FusionConfig(l_c=l_c, passes=True))
                assert bits_equal(st.to_numpy(), want), (build.__name__, l_c)


def test_passes_records_and_golden(golden):
    d = golden("circuits_small")
    from conftest import golden_circuit

    for name, n in (("mix10", 10), ("ctl12", 12)):
        circ = golden_circuit(d, name, n)
        st = sv.state_from_global(sv.Layout(n), d[f"{name}_in"], device=DEV)
        recs = sv.run_circuit(st, circ, fusion=sv.FusionConfig(l_c=13, passes=True), record=True)
        assert np.array_equal(st.to_numpy(), d[f"{name}_out"])
        assert sum(r.gate_count for r in recs) == len(circ)
        assert all(r.seconds > 0 for r in recs)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_loopback_global_stages_bitwise(p):
    """Transform stages on global targets: one exchange per stage, bits equal to the oracle."""
    n = 14
    rng = np.random.default_rng(300 + p)
    v = with_zeros(rng, n)
    circ = sv.build_qft(n)
    circ.extend(random_ops(rng, n, 40, n))
    want = run_oracle(v, circ.gates)
    got, _ = run_loopback(n, p, circ, v, fusion=sv.FusionConfig(l_c=9, passes=True))
    assert bits_equal(got, want)


def test_exchange_stage_abi_guards():
    from paper_1601_07195_b200 import _lib

    a = torch.zeros(64, dtype=torch.complex128, device=DEV)
    b = torch.zeros(64, dtype=torch.complex128, device=DEV)
    g = sv.kernels.gate_array([sv.GateOp(sv.hadamard(), 6, 7)])
    st = torch.cuda.current_stream().cuda_stream
    L = _lib.load()
    assert L.sv_exchange_stage(a.data_ptr(), b.data_ptr(), 6, 1, g, 1, st) == _lib.SV_EINVAL  # control 7 not local
    assert L.sv_exchange_stage(a.data_ptr(), b.data_ptr(), 6, 1, g, 0, st) == _lib.SV_EINVAL
    assert L.sv_apply_gates(a.data_ptr(), 6, g, 1, 0, st) == _lib.SV_EINVAL  # target 6 not local


@pytest.mark.parametrize("slots", [2, 3])
def test_run_pipelined_matches_run_circuit(slots):
    n = 16
    rng = np.random.default_rng(44)
    circs = [sv.random_circuit(n, 30, rng, controlled_fraction=0.4) for _ in range(5)]
    ins = [torch.from_numpy(random_state(rng, n)).pin_memory() for _ in range(5)]
    outs = [torch.empty_like(x).pin_memory() for x in ins]
    sv.run_pipelined(sv.Layout(n), circs, ins, outs, fusion=sv.FusionConfig(l_c=12, passes=True), slots=slots)
    torch.cuda.synchronize()
    for c, x, y in zip(circs, ins, outs):
        want = run_oracle(x.numpy(), c.gates)
        assert bits_equal(y.numpy(), want)


def test_circuit_graph_replay_bitwise():
    n = 20
    rng = np.random.default_rng(45)
    v = random_state(rng, n)
    circ = sv.random_circuit(n, 60, rng, controlled_fraction=0.3)
    st = sv.state_from_global(sv.Layout(n), v, device=DEV)
    g = sv.CircuitGraph(st, circ, fusion=sv.FusionConfig(l_c=13, passes=True))
    g.replay()
    g.replay()
    want = run_oracle(run_oracle(v, circ.gates), circ.gates)
    assert bits_equal(st.to_numpy(), want)


@pytest.mark.parametrize("n", [13, 17])
def test_speculative_paths_replay_exactly_on_zeros(n):
    """Diagonal/phase-dominated runs take the speculative kernels; states salted with +-0 and
    'nice' values force the exact replay -- bits must still equal the oracle."""
    rng = np.random.default_rng(900 + n)
    diag = [sv.phase_r(2), sv.phase_r(5).dagger(), sv.pauli_z(), sv.rotation_z(0.7),
            sv.GateMatrix([[1j, 0], [0, -1]]), sv.GateMatrix.unchecked([[1, -0.0], [0.0, 1j]])]
    for trial in range(4):
        v = with_zeros(rng, n, frac=0.3) if trial % 2 else np.full(1 << n, 2.0 ** (-n / 2), dtype=np.complex128)
        ops = []
        for _ in range(80):
            t = int(rng.integers(n if trial < 2 else 12))
            c = None if rng.random() < 0.3 else int((t + 1 + rng.integers(n - 1)) % n)
            ops.append(sv.GateOp(diag[int(rng.integers(len(diag)))], t, c))
        ops.insert(0, sv.GateOp(sv.hadamard(), n - 1))
        a = torch.from_numpy(v.copy()).to(DEV)
        sv.kernels.apply_gates(a, ops)
        torch.cuda.synchronize()
        assert bits_equal(a.cpu().numpy(), run_oracle(v, ops)), trial


@pytest.mark.parametrize("n", [13, 16])
def test_speculation_tests_only_the_final_values(n):
    """The fused kernels test for zeros once, after the whole run (a dropped zero term of mix()
    can only flip the sign of a zero).  Exact cancellations in the MIDDLE of a phase chain
    -- (0.5+0.5j) * (0.5+0.5j) has real part exactly 0 -- must not change a bit whether the zero
    survives to the end (replay) or is rotated away by the next phase (no replay)."""
    rng = np.random.default_rng(77 + n)
    cancel = sv.GateMatrix.unchecked([[1, 0], [0, 0.5 + 0.5j]])
    rot = [sv.phase_r(3), sv.rotation_z(0.3), sv.pauli_z(), sv.GateMatrix.unchecked([[1, 0], [0, 1j]])]
    v = np.full(1 << n, 0.5 + 0.5j, dtype=np.complex128)
    for trial in range(3):
        ops = []
        for _ in range(60):
            t = int(rng.integers(n if trial == 0 else (12 if trial == 1 else n - 1)))
            if trial == 2:
                t = n - 1  # one same-target stage
            c = None if rng.random() < 0.4 else int((t + 1 + rng.integers(n - 1)) % n)
            g = cancel if rng.random() < 0.4 else rot[int(rng.integers(len(rot)))]
            ops.append(sv.GateOp(g, t, c))
        if trial == 2:
            ops.insert(0, sv.GateOp(sv.hadamard(), n - 1))
        a = torch.from_numpy(v.copy()).to(DEV)
        sv.kernels.apply_gates(a, ops)
        torch.cuda.synchronize()
        assert bits_equal(a.cpu().numpy(), run_oracle(v, ops)), trial
