"""Edge cases through the C ABI: tiny registers, every kernel path at its smallest size,
fused runs below the register-tile limit, exchanges at m = 1..4, host I/O round trips."""

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


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6])
def test_tiny_registers_every_gate(n):
    rng = np.random.default_rng(n)
    v = random_state(rng, n)
    ops = [sv.GateOp(sv.random_unitary(rng), k) for k in range(n)]
    ops += [sv.GateOp(sv.random_unitary(rng), t, c) for c in range(n) for t in range(n) if c != t]
    want = v.copy()
    oracle.run_circuit(want, ops)
    circ = sv.Circuit(n, ops)
    for fusion in (None, sv.FusionConfig(l_c=n), sv.FusionConfig(l_c=max(1, n - 1)),
                   sv.FusionConfig(l_c=n, passes=True)):
        st = sv.state_from_global(sv.Layout(n), v, device=DEV)
        sv.run_circuit(st, circ, fusion=fusion)
        assert np.array_equal(bits(st.to_numpy()), bits(want)), fusion


@pytest.mark.parametrize("n,p", [(2, 1), (3, 1), (3, 2), (4, 3), (5, 2)])
def test_exchange_smallest_slices(n, p):
    rng = np.random.default_rng(10 * n + p)
    v = random_state(rng, n)
    ops = [sv.GateOp(sv.random_unitary(rng), k) for k in range(n)]
    ops += [sv.GateOp(sv.random_unitary(rng), t, c) for c in range(n) for t in range(n) if c != t]
    want = v.copy()
    oracle.run_circuit(want, ops)
    circ = sv.Circuit(n, ops)
    got, _ = run_loopback(n, p, circ, v)
    assert np.array_equal(bits(got), bits(want))
    got2, _ = run_loopback(n, p, circ, v, fusion=sv.FusionConfig(l_c=n - p, passes=True))
    assert np.array_equal(bits(got2), bits(want))


def test_empty_and_single_gate_circuits():
    n = 8
    v = random_state(np.random.default_rng(3), n)
    st = sv.state_from_global(sv.Layout(n), v, device=DEV)
    assert sv.run_circuit(st, sv.Circuit(n)) is None
    assert sv.run_circuit(st, sv.Circuit(n), record=True) == []
    sv.kernels.apply_gates(st.amps, [])
    assert np.array_equal(st.to_numpy(), v)
    q = sv.random_unitary(np.random.default_rng(4))
    sv.run_circuit(st, sv.Circuit(n, [sv.GateOp(q, 7)]), fusion=sv.FusionConfig(l_c=8, passes=True))
    want = v.copy()
    oracle.apply_single(want, 7, q)
    assert np.array_equal(st.to_numpy(), want)


def test_host_io_round_trip_and_guards():
    n = 12
    v = random_state(np.random.default_rng(5), n)
    st = sv.state_from_global(sv.Layout(n), v, device=DEV)
    h = torch.empty(1 << n, dtype=torch.complex128).pin_memory()
    st.store_host(h)
    torch.cuda.synchronize()
    assert np.array_equal(h.numpy(), v)
    h2 = torch.from_numpy(random_state(np.random.default_rng(6), n)).pin_memory()
    st.load_host(h2)
    torch.cuda.synchronize()
    assert np.array_equal(st.to_numpy(), h2.numpy())
    with pytest.raises(sv.LayoutError):
        st.load_host(torch.empty(8, dtype=torch.complex128))
    with pytest.raises(TypeError):
        st.load_host(torch.empty(1 << n, dtype=torch.complex128, device=DEV))


def test_basis_states_and_probabilities_sharded():
    n, p = 9, 2
    for basis in (0, 5, 300, 511):
        full = []
        for r in range(1 << p):
            s = sv.init_basis_state(sv.Layout(n, p, r), basis, device=DEV)
            full.append(s.to_numpy())
        f = np.concatenate(full)
        assert f[basis] == 1.0 and np.count_nonzero(f) == 1
    st = sv.state_from_global(sv.Layout(6), random_state(np.random.default_rng(7), 6), device=DEV)
    a = st.to_numpy()
    for b in range(6):
        want = float(np.sum(np.abs(a.reshape(-1, 2, 1 << b)[:, 1, :]) ** 2))
        assert abs(sv.probability_of_bit(st, b) - want) < 1e-14
    with pytest.raises(ValueError):
        sv.probability_of_bit(st, 6)


def test_max_abs_diff_kernel():
    """sv_max_abs_diff (the bench self-check) against numpy, including a single far element."""
    rng = np.random.default_rng(5)
    for n in (0, 3, 10, 17):
        a = random_state(rng, n) if n else np.array([0.3 + 0.4j])
        b = a + (rng.standard_normal(a.shape) + 1j * rng.standard_normal(a.shape)) * 1e-9
        b[-1] += 0.25j
        want = float(np.max(np.abs(a - b)))
        got = sv.max_abs_diff(torch.from_numpy(a).to(DEV), torch.from_numpy(b).to(DEV))
        assert got == pytest.approx(want, rel=1e-15, abs=0)


def test_raw_kernels_accept_strided_views():
    """The reference's *_raw kernels work on uniformly strided numpy views (kernels.py:174-184);
    here a strided 1-D CUDA view is updated through a contiguous copy, bit for bit."""
    import torch

    from oracle import oracle

    rng = np.random.default_rng(8)
    base = rng.standard_normal(512) + 1j * rng.standard_normal(512)
    dev = torch.from_numpy(base.copy()).to("cuda:0")
    view = dev[1::2]
    want = base.copy()
    q1, q2 = sv.random_unitary(rng), sv.random_unitary(rng)
    w = want[1::2].copy()
    oracle.apply_single(w, 4, q1.mat)
    oracle.apply_controlled(w, 0, 7, q2.mat)
    want[1::2] = w
    sv.apply_single_raw(view, 4, q1)
    sv.apply_controlled_raw(view, 0, 7, q2)
    torch.cuda.synchronize()
    assert np.array_equal(dev.cpu().numpy(), want)
