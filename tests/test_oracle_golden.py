"""Pin the oracle: bit-for-bit against vectors produced by the reference itself (tests/golden/).

CPU only.  If these pass, the oracle restates the reference's arithmetic
exactly, so GPU == oracle (test_gpu_parity) means GPU == reference.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import max_abs_diff, random_state, unpack_ops
from oracle import oracle


def test_kernels_n5_bitwise(golden):
    d = golden("kernels_n5")
    for inp, q, out, (c, t) in zip(d["inp"], d["q"], d["out"], d["ct"]):
        w = inp.copy()
        if c < 0:
            oracle.apply_single(w, int(t), q.reshape(2, 2))
        else:
            oracle.apply_controlled(w, int(c), int(t), q.reshape(2, 2))
        assert np.array_equal(w, out), (c, t)


@pytest.mark.parametrize("name", ["mix8", "mix10", "ctl12", "single12"])
def test_circuits_bitwise_unfused_fused_distributed(golden, name):
    d = golden("circuits_small")
    ops = unpack_ops(d, name)
    for threads in (1, 3):
        w = d[f"{name}_in"].copy()
        oracle.run_circuit(w, ops, threads=threads)
        assert np.array_equal(w, d[f"{name}_out"])
    # the reference's fused and distributed runs are bitwise equal to serial
    for key in ("fused3", "fused6", "p1", "p2", "p3"):
        assert np.array_equal(d[f"{name}_{key}"], d[f"{name}_out"]), key


def test_block_run_equals_serial(golden):
    d = golden("circuits_small")
    ops = unpack_ops(d, "mix10")
    for l in (3, 5, 9):
        w = d["mix10_in"].copy()
        low = [op for op in ops if max(op[0], -1 if op[1] is None else op[1]) < l]
        oracle.apply_block_run(w, l, low, threads=2)
        want = d["mix10_in"].copy()
        oracle.run_circuit(want, low)
        assert np.array_equal(w, want)


def test_exchange_restatement_equals_serial(golden):
    """or_exchange over rank slices (both halves) == the reference's distributed output."""
    d = golden("circuits_small")
    n = 10
    ops = unpack_ops(d, "mix10")
    for p in (1, 2, 3):
        m = n - p
        slices = [d["mix10_in"][r << m:(r + 1) << m].copy() for r in range(1 << p)]
        for t, c, q in ops:
            for r in range(1 << p):
                mine = slices[r]
                if c is None and t < m:
                    oracle.apply_single(mine, t, q)
                elif c is not None and c < m and t < m:
                    oracle.apply_controlled(mine, c, t, q)
                elif c is not None and t < m:  # remote control
                    if (r >> (c - m)) & 1:
                        oracle.apply_single(mine, t, q)
                elif c is not None and c >= m and not (r >> (c - m)) & 1:
                    pass
                else:
                    partner = r ^ (1 << (t - m))
                    zero = not (r >> (t - m)) & 1
                    oracle.exchange(mine, slices[partner], zero, -1 if c is None or c >= m else c, q)
        assert np.array_equal(np.concatenate(slices), d["mix10_p%d" % p]), p


def test_transforms_bitwise_and_closed_form(golden):
    d = golden("transforms")
    for n in (10, 12):
        for name in ("qft", "iqft"):
            w = d[f"{name}{n}_in"].copy()
            oracle.run_circuit(w, unpack_ops(d, f"{name}{n}"))
            assert np.array_equal(w, d[f"{name}{n}_out"])
    assert max_abs_diff(d["qft8_basis5"], oracle.dft_bit_reversed(8, 5)) <= 1e-12


def test_config1_sample_bitwise(golden):
    """Full BASELINE config 1 through the oracle: sampled amplitudes + hash equal the reference's."""
    import hashlib

    d = golden("config1_n20")
    n = int(d["n"])
    rng0 = np.random.default_rng(0)
    raw = rng0.standard_normal(1 << n) + 1j * rng0.standard_normal(1 << n)
    init = (raw / float(d["norm"])).astype(np.complex128)
    assert hashlib.sha256(init.tobytes()).hexdigest() == str(d["in_sha"])
    ops = [(int(t), None, q.reshape(2, 2)) for t, q in zip(d["t"], d["q"])]
    oracle.run_circuit(init, ops, threads=8)
    assert np.array_equal(init[d["idx"]], d["out_sample"])
    assert hashlib.sha256(init.tobytes()).hexdigest() == str(d["out_sha"])


def test_dense_oracle_cross_check(rng):
    """Index-free Kronecker restatement agrees with the strided oracle to 1e-13 (test_kernels.py:52-76)."""
    import paper_1601_07195_b200 as sv

    n = 5
    q = sv.random_unitary(rng)
    for k in range(n):
        v = random_state(rng, n)
        w = v.copy()
        oracle.apply_single(w, k, q)
        assert max_abs_diff(w, oracle.dense_single(n, k, q) @ v) < 1e-13
    for c in range(n):
        for t in range(n):
            if c != t:
                v = random_state(rng, n)
                w = v.copy()
                oracle.apply_controlled(w, c, t, q)
                assert max_abs_diff(w, oracle.dense_controlled(n, c, t, q) @ v) < 1e-13


def test_norm_and_probabilities(golden):
    d = golden("known_answers")
    st = d["prob_state"]
    assert abs(oracle.norm_sq(st) - float(d["prob_norm"])) < 1e-13
    for b in range(6):
        assert abs(oracle.norm_sq(st, b) - d["prob_bits"][b]) < 1e-13
    for g in range(4):
        v = np.zeros(4, complex)
        v[g] = 1.0
        oracle.apply_controlled(v, 0, 1, np.array([[0, 1], [1, 0]], complex))
        assert np.array_equal(v, d[f"cnot_{g}"])
