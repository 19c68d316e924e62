"""Local gate entry points, B200 edition of pkg/src/svsim/kernels.py.

Same names, signatures, in-place semantics and exception classes as the
reference; the work is one launch of a hand-written sm_100a kernel through
the C ABI (include/svb200.h) on the caller's current CUDA stream:

* ``apply_single_raw``      kernels.py:187-189  -> ``sv_apply_single``
* ``apply_controlled_raw``  kernels.py:192-196  -> ``sv_apply_controlled``
* ``apply_single_local``    kernels.py:199-208  (LayoutError guard, then raw)
* ``apply_controlled_local`` kernels.py:211-222 (ValueError / LayoutError guards)
* ``apply_block``           kernels.py:225-240  -> ``sv_apply_fused`` on one block

``ThreadPolicy`` is accepted for signature compatibility and ignored: the
CUDA grid replaces the reference's OUTER/INNER loop split (kernels.py:77-171),
and results are bitwise independent of it, as the reference guarantees for
its own split.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass
from typing import TYPE_CHECKING, Iterable

import numpy as np
import torch

from . import _lib
from .errors import FusionContractError, LayoutError

if TYPE_CHECKING:
    from .circuits import GateOp
    from .core import LocalState

UNITARITY_TOL = 1e-12


class GateMatrix:
    """Read-only 2x2 complex matrix; unitarity checked to 1e-12 unless `unchecked`.

    Reference: kernels.py:36-74.  The matrix lives on the host; each launch
    passes its 8 doubles by value as a kernel parameter.
    """

    __slots__ = ("mat", "_q")

    def __init__(self, mat, check: bool = True):
        arr = np.array(mat, dtype=np.complex128).reshape(2, 2)
        if check:
            dev = float(np.max(np.abs(arr.conj().T @ arr - np.eye(2))))
            if dev > UNITARITY_TOL:
                raise ValueError(f"matrix is not unitary (deviation {dev:.2e})")
        arr.flags.writeable = False
        self.mat = arr
        self._q = None

    @classmethod
    def unchecked(cls, mat) -> "GateMatrix":
        return cls(mat, check=False)

    @property
    def q11(self) -> complex:
        return complex(self.mat[0, 0])

    @property
    def q12(self) -> complex:
        return complex(self.mat[0, 1])

    @property
    def q21(self) -> complex:
        return complex(self.mat[1, 0])

    @property
    def q22(self) -> complex:
        return complex(self.mat[1, 1])

    def dagger(self) -> "GateMatrix":
        return GateMatrix.unchecked(self.mat.conj().T)

    def qbuf(self):
        """The 8-double ABI form, cached (the matrix is immutable)."""
        if self._q is None:
            self._q = _lib.qbuf(self.mat)
        return self._q

    def __repr__(self) -> str:
        return f"GateMatrix({self.mat.tolist()})"


class ParallelLevel(enum.Enum):
    OUTER = "outer"
    INNER = "inner"
    AUTO = "auto"


@dataclass(frozen=True)
class ThreadPolicy:
    """Signature-compatible stand-in for the reference's CPU loop split."""

    num_threads: int = 1
    parallel_level: ParallelLevel = ParallelLevel.AUTO

    def __post_init__(self):
        if self.num_threads < 1:
            raise ValueError("num_threads must be >= 1")

    def resolve(self, outer_iters: int) -> ParallelLevel:
        if self.parallel_level is not ParallelLevel.AUTO:
            return self.parallel_level
        return ParallelLevel.OUTER if outer_iters >= self.num_threads else ParallelLevel.INNER


SERIAL = ThreadPolicy(1)


def _as_gate(q) -> GateMatrix:
    return q if isinstance(q, GateMatrix) else GateMatrix.unchecked(q)


def stream_handle() -> int:
    """cudaStream_t of torch's current stream on the current device."""
    return torch.cuda.current_stream().cuda_stream


def device_view(amps) -> tuple[int, int]:
    """(device pointer, m) of a contiguous complex128 CUDA vector of 2^m elements."""
    if not isinstance(amps, torch.Tensor):
        raise TypeError("amplitudes must be a torch complex128 CUDA tensor (no host path)")
    if amps.dtype != torch.complex128:
        raise TypeError("amplitudes must be complex128")
    if not amps.is_cuda:
        raise TypeError("amplitudes must live on a CUDA device (there is no CPU fallback)")
    if amps.dim() != 1 or not amps.is_contiguous():
        raise ValueError("amplitudes must be a contiguous 1-D vector")
    n = amps.shape[0]
    m = n.bit_length() - 1
    if n < 1 or n != 1 << m:
        raise ValueError(f"cannot view {n} amplitudes as a qubit register (need a power of two)")
    return amps.data_ptr(), m


def _strided(amps, fn) -> bool:
    """A uniformly strided 1-D CUDA view (what the reference's reshape views are): run `fn` on
    a contiguous copy and write the result back.  Returns False for contiguous inputs."""
    if isinstance(amps, torch.Tensor) and amps.is_cuda and amps.dim() == 1 and not amps.is_contiguous():
        tmp = amps.contiguous()
        fn(tmp)
        amps.copy_(tmp)
        return True
    return False


def apply_single_raw(amps, k: int, q, policy: ThreadPolicy = SERIAL) -> None:
    """In-place single-qubit update on bit k (kernels.py:187-189); no layout checks.
    Uniformly strided 1-D views are accepted (copy-in / copy-out), as the reference's are."""
    if _strided(amps, lambda t: apply_single_raw(t, k, q, policy)):
        return
    ptr, m = device_view(amps)
    if not 0 <= k < m:
        raise ValueError(f"qubit {k} out of range for a {m}-qubit slice")
    with torch.cuda.device(amps.device):
        _lib.check(_lib.load().sv_apply_single(ptr, m, int(k), _as_gate(q).qbuf(), stream_handle()))


def apply_controlled_raw(amps, c: int, t: int, q, policy: ThreadPolicy = SERIAL) -> None:
    """In-place controlled update, control c / target t (kernels.py:192-196); strided views as above."""
    if _strided(amps, lambda a: apply_controlled_raw(a, c, t, q, policy)):
        return
    ptr, m = device_view(amps)
    if c == t:
        raise ValueError(f"control and target must differ, both are {c}")
    if not (0 <= c < m and 0 <= t < m):
        raise ValueError(f"qubits ({c},{t}) out of range for a {m}-qubit slice")
    with torch.cuda.device(amps.device):
        _lib.check(_lib.load().sv_apply_controlled(ptr, m, int(c), int(t), _as_gate(q).qbuf(),
                                                   stream_handle()))


def apply_single_local(state: "LocalState", k: int, q: GateMatrix, policy: ThreadPolicy = SERIAL) -> None:
    """Single-qubit gate on local qubit k < m, in place (kernels.py:199-208)."""
    m = state.layout.m
    if not 0 <= k < m:
        raise LayoutError(
            f"qubit {k} is not local (m={m}); gates on qubits >= m need the distributed path"
        )
    apply_single_raw(state.amps, k, q, policy)


def apply_controlled_local(
    state: "LocalState", c: int, t: int, q: GateMatrix, policy: ThreadPolicy = SERIAL
) -> None:
    """Controlled gate with both qubits local, in place (kernels.py:211-222)."""
    if c == t:
        raise ValueError(f"control and target must differ, both are {c}")
    m = state.layout.m
    if c >= m or t >= m or c < 0 or t < 0:
        raise LayoutError(f"qubits ({c},{t}) are not both local (m={m}); use the distributed path")
    apply_controlled_raw(state.amps, c, t, q, policy)


def gate_array(ops):
    """ctypes array of sv_gate for a sequence of GateOp."""
    ops = list(ops)
    arr = (_lib.SvGate * max(1, len(ops)))()
    for i, op in enumerate(ops):
        arr[i].target = op.target
        arr[i].control = -1 if op.control is None else op.control
        arr[i].q[:] = list(_as_gate(op.gate).qbuf())
    return arr


def launch_fused(amps, ops: list, l: int) -> None:
    """sv_apply_fused over every 2^l block of `amps` (caller validated the run)."""
    ptr, m = device_view(amps)
    lib = _lib.load()
    with torch.cuda.device(amps.device):
        for lo in range(0, len(ops), _lib.SV_FUSED_MAX_GATES):
            part = ops[lo:lo + _lib.SV_FUSED_MAX_GATES]
            _lib.check(lib.sv_apply_fused(ptr, m, int(l), gate_array(part), len(part), stream_handle()))


def apply_gates(amps, ops, tile: int = 0, exact: bool = True) -> None:
    """Native pass planner (sv_apply_gates): local gates applied in order, grouped into
    register-tiled runs (targets < tile, controls anywhere) and multi-target stage passes
    (runs whose targets lie in at most four qubits).
    Bit-identical to applying them one by one; exact=False: the tolerance mode
    (SV_FLAG_TOLERANCE, equal within rounding)."""
    ptr, m = device_view(amps)
    ops = list(ops)
    if not ops:
        return
    for op in ops:
        if op.max_qubit() >= m:
            raise LayoutError(f"gate on qubits {op.qubits()} is not local (m={m})")
    with torch.cuda.device(amps.device):
        _lib.check(_lib.load().sv_apply_gates_ex(ptr, m, gate_array(ops), len(ops), int(tile),
                                                 0 if exact else _lib.SV_FLAG_TOLERANCE, stream_handle()))


def apply_block(block_amps, gates: Iterable["GateOp"], policy: ThreadPolicy = SERIAL) -> None:
    """Apply gates in order to one contiguous 2^b slice as a b-qubit state (kernels.py:225-240).

    Runs as one shared-memory-resident tile pass when b <= SV_FUSED_MAX_TILE;
    larger blocks fall back to per-gate passes of the local kernels (same
    arithmetic, so the result is identical).
    """
    ops = list(gates)
    _, b = device_view(block_amps)
    for op in ops:
        if op.max_qubit() >= b:
            raise FusionContractError(f"gate on qubits {op.qubits()} exceeds block exponent {b}")
    if not ops:
        return
    if b <= _lib.SV_FUSED_MAX_TILE:
        launch_fused(block_amps, ops, b)
        return
    for op in ops:
        if op.control is None:
            apply_single_raw(block_amps, op.target, op.gate, policy)
        else:
            apply_controlled_raw(block_amps, op.control, op.target, op.gate, policy)
