"""Global<->local qubit remapping: the swap plan, checked on CPU by
emulating it on a full state vector -- swaps as bit permutations of the index, physical
gates through the oracle -- against the oracle on the logical circuit, bit for bit."""

from __future__ import annotations

import numpy as np
import pytest

import paper_1601_07195_b200 as sv
from conftest import random_state
from oracle import oracle


def swap_bits(v, a, b):
    n = v.shape[0].bit_length() - 1
    t = v.reshape((2,) * n)  # axis k <-> bit n-1-k
    return np.ascontiguousarray(np.swapaxes(t, n - 1 - a, n - 1 - b)).reshape(-1)


def emulate(v, items):
    w = v.copy()
    for it in items:
        if isinstance(it, sv.Swap):
            w = swap_bits(w, it.global_bit, it.local_bit)
        else:
            oracle.run_circuit(w, it)
    return w


@pytest.mark.parametrize("n,p,seed", [(8, 1, 0), (9, 2, 1), (10, 3, 2), (11, 2, 3), (12, 3, 4)])
def test_plan_reproduces_the_circuit_bitwise(n, p, seed):
    m = n - p
    rng = np.random.default_rng(seed)
    circ = sv.random_circuit(n, 120, rng, controlled_fraction=0.4)
    circ.extend(sv.build_qft(n).gates)
    v = random_state(rng, n)
    want = v.copy()
    oracle.run_circuit(want, circ.gates)
    items, qm = sv.plan_remapped(circ.gates, n, m)
    assert qm.identity
    for it in items:
        if isinstance(it, sv.Swap):
            assert m <= it.global_bit < n and 0 <= it.local_bit < m
        else:
            assert all(op.target < m for op in it)  # every gate runs locally
    got = emulate(v, items)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    # fewer link bytes than the in-place exchanges: swaps move half as much
    n_exch = sum(1 for op in circ if op.target >= m)
    n_swap = sum(isinstance(it, sv.Swap) for it in items)
    assert n_swap <= 2 * n_exch


def test_unrestored_map_and_continuation():
    n, m = 9, 7
    rng = np.random.default_rng(9)
    a = sv.random_circuit(n, 40, rng)
    b = sv.random_circuit(n, 40, rng)
    v = random_state(rng, n)
    want = v.copy()
    oracle.run_circuit(want, a.gates + b.gates)
    items1, qm = sv.plan_remapped(a.gates, n, m, restore=False)
    w = emulate(v, items1)
    items2, qm = sv.plan_remapped(b.gates, n, m, restore=True, qmap=qm)
    w = emulate(w, items2)
    assert qm.identity and np.array_equal(w.view(np.uint64), want.view(np.uint64))


def test_link_traffic_of_the_baseline_circuits():
    """Swaps (half an exchange each) against in-place exchanges: a per-target sweep brings
    each global qubit in and one victim back per visit (2g swaps per sweep: no saving); the
    transform needs six swaps at g = 3 instead of 99 exchanges."""
    n, m = 12, 9
    circ = sv.per_target_sweep(n, 3, np.random.default_rng(0))
    items, qm = sv.plan_remapped(circ.gates, n, m)
    swaps = [it for it in items if isinstance(it, sv.Swap)]
    assert qm.identity and len(swaps) <= 2 * 3 * (n - m) + (n - m)
    items, qm = sv.plan_remapped(sv.build_qft(34).gates, 34, 31)
    assert sum(isinstance(it, sv.Swap) for it in items) == 6
    circ = sv.random_circuit(36, 100, np.random.default_rng(1), controlled_fraction=0.0)
    items, _ = sv.plan_remapped(circ.gates, 36, 33)
    assert sum(isinstance(it, sv.Swap) for it in items) <= sum(op.target >= 33 for op in circ)


def test_more_global_than_local_qubits_falls_back_to_exchanges():
    n, m = 6, 2  # four global qubits, two local
    rng = np.random.default_rng(12)
    circ = sv.random_circuit(n, 80, rng, controlled_fraction=0.3)
    v = random_state(rng, n)
    want = v.copy()
    oracle.run_circuit(want, circ.gates)
    items, qm = sv.plan_remapped(circ.gates, n, m)
    assert qm.identity
    # the emulation applies physical gates with the oracle, exchanges included
    got = emulate(v, items)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    assert any(op.target >= m for it in items if not isinstance(it, sv.Swap) for op in it)
