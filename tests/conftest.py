"""Shared fixtures.  `gpu` tests need a CUDA device (run on the B200 box);
everything else runs on CPU.  The oracle (oracle/) is imported only here and
in tests, as the checker."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = dict(np.load(GOLDEN / f"{name}.npz"))
        return cache[name]

    return load


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def random_state(rng, n):
    """Reference test recipe (pkg/tests/test_kernels.py:32-34)."""
    v = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    return (v / np.linalg.norm(v)).astype(np.complex128)


def unpack_ops(d, prefix):
    """(target, control|None, 2x2) triples of a golden circuit."""
    return [(int(t), None if c < 0 else int(c), q.reshape(2, 2))
            for t, c, q in zip(d[f"{prefix}_t"], d[f"{prefix}_c"], d[f"{prefix}_q"])]


def golden_circuit(d, prefix, n):
    """A Circuit of the package built from stored golden matrices (not regenerated)."""
    import paper_1601_07195_b200 as sv

    return sv.Circuit(n, [sv.GateOp(sv.GateMatrix.unchecked(q), t, c) for t, c, q in unpack_ops(d, prefix)])


def max_abs_diff(a, b) -> float:
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))))
