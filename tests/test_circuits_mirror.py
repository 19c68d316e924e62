"""The package's circuit builders reproduce the reference's gates for the same generator state
(compared with the matrices the reference itself stored in tests/golden/)."""

from __future__ import annotations

import math

import numpy as np

import paper_1601_07195_b200 as sv


def _check(circ, d, prefix, exact=True):
    assert [op.target for op in circ] == [int(x) for x in d[f"{prefix}_t"]]
    assert [-1 if op.control is None else op.control for op in circ] == [int(x) for x in d[f"{prefix}_c"]]
    got = np.stack([op.gate.mat.reshape(4) for op in circ])
    if exact:
        assert np.array_equal(got, d[f"{prefix}_q"])
    else:  # QR goes through LAPACK, which may round differently on another CPU
        assert np.max(np.abs(got - d[f"{prefix}_q"])) < 1e-14


def test_random_circuits_match_reference(golden):
    d = golden("circuits_small")
    for name, n, g, frac, seed in (("mix10", 10, 120, 0.3, 7), ("ctl12", 12, 100, 1.0, 11),
                                   ("single12", 12, 100, 0.0, 13), ("mix8", 8, 100, 0.3, 8)):
        _check(sv.random_circuit(n, g, np.random.default_rng(seed), controlled_fraction=frac), d, name,
               exact=False)


def test_config1_circuit_matches_reference(golden):
    d = golden("config1_n20")
    circ = sv.random_circuit(20, 200, np.random.default_rng(1), controlled_fraction=0.0)
    assert [op.target for op in circ] == [int(x) for x in d["t"]]
    got = np.stack([op.gate.mat.reshape(4) for op in circ])
    assert np.max(np.abs(got - d["q"])) < 1e-14


def test_transform_builders_match_reference(golden):
    d = golden("transforms")
    for n in (10, 12):
        _check(sv.build_qft(n), d, f"qft{n}")
        _check(sv.build_iqft(n), d, f"iqft{n}")


def test_named_gates():
    assert np.allclose(sv.phase_r(1).mat, np.diag([1, -1]))
    assert np.allclose(sv.phase_r(2).mat, np.diag([1, 1j]))
    h = sv.hadamard().mat
    assert np.allclose(h @ h, np.eye(2))
    for g in (sv.pauli_x(), sv.pauli_y(), sv.pauli_z(), sv.rotation_x(0.3), sv.rotation_y(1.1),
              sv.rotation_z(-0.7)):
        assert np.allclose(g.mat.conj().T @ g.mat, np.eye(2))
    qft1 = sv.build_qft(1)
    assert len(qft1) == 1 and np.array_equal(qft1.gates[0].gate.mat, sv.hadamard().mat)
    assert math.isclose(abs(sv.rotation_z(0.4).mat[0, 0]), 1.0)


def test_inverse_and_sweep():
    circ = sv.random_circuit(6, 10, np.random.default_rng(2))
    inv = circ.inverse()
    assert [op.target for op in inv] == [op.target for op in reversed(circ.gates)]
    sweep = sv.per_target_sweep(30, 2, np.random.default_rng(1))
    assert [op.target for op in sweep] == list(range(30)) * 2
