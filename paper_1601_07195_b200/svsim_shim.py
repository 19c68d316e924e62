"""Reference-side binding: make the stock ``svsim`` package call libsvb200.

``install(svsim)`` replaces the reference's two raw kernels -- the functions every local
gate of ``svsim`` goes through (``apply_single_raw`` / ``apply_controlled_raw``,
pkg/src/svsim/kernels.py:187-196, called from kernels.py:208, :222, :238-240 and
distributed.py:382, :388) -- with ctypes calls into ``sv_apply_single`` /
``sv_apply_controlled``.  ``svsim.distributed`` binds the raw kernels by name at import
(distributed.py:29-36), so both modules are patched.  States stay numpy arrays: each call
uploads the slice, runs the kernel and downloads it (PCIe-bound; the package-level drop-in
``paper_1601_07195_b200`` keeps the state on the GPU instead).  Uniformly strided views --
which the reference's reshape views accept -- are handled by copy-in / copy-out.

The kernels reproduce numpy's rounding sequence exactly, so ``svsim``'s results are
bit-identical with and without the shim (tests/test_gpu_shim.py drives the reference's own
golden circuits through the patched package).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib

_ORIGINALS: dict = {}


def _q(gate) -> ctypes.Array:
    mat = np.asarray(getattr(gate, "mat", gate), dtype=np.complex128).reshape(4)
    return (ctypes.c_double * 8)(*np.ascontiguousarray(mat).view(np.float64).tolist())


def _run(amps: np.ndarray, call) -> None:
    if amps.dtype != np.complex128 or amps.ndim != 1:
        raise ValueError("the B200 shim needs a 1-D complex128 slice")
    n = amps.shape[0]
    m = n.bit_length() - 1
    if n < 1 or n != 1 << m:
        raise ValueError(f"cannot reshape array of size {n} into a qubit register")
    dev = torch.from_numpy(np.ascontiguousarray(amps)).to("cuda")
    rc = call(dev.data_ptr(), m, torch.cuda.current_stream().cuda_stream)
    _lib.check(rc)
    amps[...] = dev.cpu().numpy()


def apply_single_raw(amps, k, q, policy=None) -> None:
    """sv_apply_single on a numpy slice (kernels.py:187-189 semantics: ValueError on a bad k)."""
    m = amps.shape[0].bit_length() - 1
    if not 0 <= int(k) < m:
        raise ValueError(f"qubit {k} out of range for a {m}-qubit slice")
    qb = _q(q)
    _run(amps, lambda p, mm, s: _lib.load().sv_apply_single(p, mm, int(k), qb, s))


def apply_controlled_raw(amps, c, t, q, policy=None) -> None:
    """sv_apply_controlled on a numpy slice (kernels.py:192-196)."""
    m = amps.shape[0].bit_length() - 1
    if c == t:
        raise ValueError(f"control and target must differ, both are {c}")
    if not (0 <= int(c) < m and 0 <= int(t) < m):
        raise ValueError(f"qubits ({c},{t}) out of range for a {m}-qubit slice")
    qb = _q(q)
    _run(amps, lambda p, mm, s: _lib.load().sv_apply_controlled(p, mm, int(c), int(t), qb, s))


def install(svsim=None):
    """Patch svsim.kernels and svsim.distributed (idempotent); returns the svsim module."""
    if svsim is None:
        import svsim
    import importlib

    for name in ("kernels", "distributed"):
        mod = importlib.import_module(f"{svsim.__name__}.{name}")
        _ORIGINALS.setdefault(mod.__name__, (mod.apply_single_raw, mod.apply_controlled_raw))
        mod.apply_single_raw = apply_single_raw
        mod.apply_controlled_raw = apply_controlled_raw
    _lib.load()
    return svsim


def uninstall(svsim=None) -> None:
    if svsim is None:
        import svsim
    import importlib

    for name in ("kernels", "distributed"):
        mod = importlib.import_module(f"{svsim.__name__}.{name}")
        orig = _ORIGINALS.pop(mod.__name__, None)
        if orig is not None:
            mod.apply_single_raw, mod.apply_controlled_raw = orig
