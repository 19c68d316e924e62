"""BASELINE.json configs 2-5 at parity sizes: the same circuit recipes,
seeds and state recipe, scaled to sizes the oracle finishes in seconds, through every
execution mode -- per-gate, pass-fused, sharded over in-process ranks (InprocFabric: the
NVLink exchange kernels on one GPU), remapped (global<->local swaps) -- bit-identical to the
oracle.  Config 1 runs at full size in test_gpu_parity.py; the full-size configs 2-5 are
checked in every bench line by undoing each step with its inverse circuit."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import random_state
from test_gpu_passes import DEV, bits_equal

pytestmark = pytest.mark.gpu

sv = pytest.importorskip("paper_1601_07195_b200")
from oracle import oracle  # noqa: E402


def run_modes(v, circ, p, modes):
    """{mode: gathered amplitudes} for the requested execution modes."""
    n = circ.n
    m = n - p
    out = {}
    for mode in modes:
        sts = [sv.LocalState(sv.Layout(n, p, r), torch.from_numpy(v[r << m:(r + 1) << m].copy()).to(DEV))
               for r in range(1 << p)]
        fabs = sv.InprocFabric.group(sts) if p else [None]
        if mode == "gates":
            sv.run_circuit_inproc(sts, circ, fabs)
        elif mode == "passes":
            sv.run_circuit_inproc(sts, circ, fabs, fusion=sv.FusionConfig(l_c=min(12, m), passes=True))
        elif mode == "blocks":
            sv.run_circuit_inproc(sts, circ, fabs, fusion=sv.FusionConfig(l_c=min(8, m)))
        elif mode == "remap":
            assert sv.run_circuit_remapped(sts, circ, fabs).identity
        torch.cuda.synchronize()
        out[mode] = np.concatenate([s.to_numpy() for s in sts])
    return out


def check(v, circ, p, modes):
    want = v.copy()
    oracle.run_circuit(want, circ.gates, threads=8)
    for mode, got in run_modes(v, circ, p, modes).items():
        assert bits_equal(got, want), mode
    return want


def test_config2_sweep_shape():
    """Per-target sweep, fresh Haar gate on every k, 10 repetitions (config 2 at n = 20)."""
    n = 20
    v = random_state(np.random.default_rng(0), n)
    circ = sv.per_target_sweep(n, 10, np.random.default_rng(1))
    check(v, circ, 0, ["gates", "passes", "blocks"])
    check(v, circ, 2, ["gates", "passes", "remap"])


def test_config3_controlled_shape():
    """300 controlled Haar gates, (c, t) uniform distinct (config 3 at n = 20)."""
    n = 20
    v = random_state(np.random.default_rng(0), n)
    circ = sv.random_circuit(n, 300, np.random.default_rng(1), controlled_fraction=1.0)
    check(v, circ, 0, ["gates", "passes"])
    check(v, circ, 1, ["gates", "passes", "remap"])


def test_config4_global_qubits_shape():
    """100 Haar gates, targets uniform over all qubits, 3 global qubits (config 4 at n = 24)."""
    n, p = 24, 3
    v = random_state(np.random.default_rng(0), n)
    circ = sv.random_circuit(n, 100, np.random.default_rng(1), controlled_fraction=0.0)
    assert sum(op.target >= n - p for op in circ) > 0
    check(v, circ, p, ["gates", "passes", "remap"])


@pytest.mark.parametrize("p", [1, 2, 3])
def test_config5_transform_shape(p):
    """build_qft on a seeded random state, mixed fused low-qubit and global-qubit gates (config 5
    at n = 22); on a basis input against the closed-form bit-reversed DFT."""
    n = 22
    v = random_state(np.random.default_rng(0), n)
    circ = sv.build_qft(n)
    check(v, circ, p, ["gates", "passes", "remap"])
    j = 123457
    basis = np.zeros(1 << n, dtype=np.complex128)
    basis[j] = 1.0
    got = run_modes(basis, circ, p, ["passes"])["passes"]
    k = np.arange(1 << n)
    rev = np.zeros_like(k)
    for b in range(n):
        rev |= ((k >> b) & 1) << (n - 1 - b)
    dft = np.exp(2j * np.pi * j * rev / 2.0 ** n) / 2.0 ** (n / 2)
    assert np.max(np.abs(got - dft)) <= 1e-12 * np.sqrt(len(circ))
