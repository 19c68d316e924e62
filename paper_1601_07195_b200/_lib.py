"""ctypes binding of libsvb200.so (include/svb200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_1601_07195_b200.build``).  There is no fallback: if the
library or a CUDA device is missing, every gate entry point raises.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libsvb200.so"

SV_OK = 0
SV_EINVAL = -1
SV_ECUDA = -2
SV_FUSED_MAX_TILE = 13
SV_FUSED_MAX_GATES = 256
SV_NORM_SCRATCH = 1025
SV_STAGE_MAX_GATES = 64
SV_MSTAGE_MAX_GATES, SV_MSTAGE_MAX_TARGETS = 128, 4
SV_TILE_GATHER = 8
SV_GROUP_GATES, SV_GROUP_TILE, SV_GROUP_STAGE, SV_GROUP_LOW, SV_GROUP_STAGE2 = 0, 1, 2, 3, 4
SV_FLAG_TOLERANCE = 1
SV_SHAPE_INTERPRETED, SV_SHAPE_FORWARD, SV_SHAPE_INVERSE = 0, 1, 2
ABI_VERSION = 1

EXPORTS = (
    "sv_version", "sv_last_error", "sv_launch_count", "sv_apply_single", "sv_apply_controlled",
    "sv_apply_fused", "sv_apply_gates", "sv_plan_gates", "sv_apply_group", "sv_exchange", "sv_exchange_chunk",
    "sv_exchange_stage", "sv_norm_sq", "sv_init_random", "sv_scale", "sv_init_basis",
    "sv_copy", "sv_ipc_handle", "sv_ipc_open", "sv_ipc_close", "sv_diag_global", "sv_diag_fix",
    "sv_swap_global", "sv_max_abs_diff", "sv_apply_gates_ex", "sv_plan_gates_ex", "sv_apply_group_ex",
    "sv_pair_update", "sv_stage2_shape", "sv_stage_shape",
)


class SvGate(ctypes.Structure):
    """sv_gate of include/svb200.h."""

    _fields_ = [("target", ctypes.c_int32), ("control", ctypes.c_int32), ("q", ctypes.c_double * 8)]


class NativeError(RuntimeError):
    """A CUDA-side failure reported by libsvb200 (SV_ECUDA)."""


_lib: ctypes.CDLL | None = None


def load() -> ctypes.CDLL:
    """Load and type the library once; raise loudly when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the gate kernels)"
        )
    L = ctypes.CDLL(str(LIB_PATH))
    vp, i, dp = ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_double)
    u64, i64 = ctypes.c_uint64, ctypes.c_int64
    sig = {
        "sv_version": ([], i),
        "sv_last_error": ([], ctypes.c_char_p),
        "sv_launch_count": ([], u64),
        "sv_apply_single": ([vp, i, i, dp, vp], i),
        "sv_apply_controlled": ([vp, i, i, i, dp, vp], i),
        "sv_apply_fused": ([vp, i, i, ctypes.POINTER(SvGate), i, vp], i),
        "sv_apply_gates": ([vp, i, ctypes.POINTER(SvGate), i, i, vp], i),
        "sv_plan_gates": ([i, ctypes.POINTER(SvGate), i, i, ctypes.POINTER(ctypes.c_int32),
                           ctypes.POINTER(ctypes.c_int32), i], i),
        "sv_apply_group": ([vp, i, i, ctypes.POINTER(SvGate), i, i, vp], i),
        "sv_apply_gates_ex": ([vp, i, ctypes.POINTER(SvGate), i, i, i, vp], i),
        "sv_plan_gates_ex": ([i, ctypes.POINTER(SvGate), i, i, i, ctypes.POINTER(ctypes.c_int32),
                              ctypes.POINTER(ctypes.c_int32), i], i),
        "sv_apply_group_ex": ([vp, i, i, ctypes.POINTER(SvGate), i, i, i, vp], i),
        "sv_stage2_shape": ([i, ctypes.POINTER(SvGate), i], i),
        "sv_stage_shape": ([i, ctypes.POINTER(SvGate), i], i),
        "sv_exchange": ([vp, vp, i, i, i, dp, vp], i),
        "sv_exchange_chunk": ([vp, vp, i, i, i, dp, u64, u64, vp], i),
        "sv_pair_update": ([vp, vp, u64, i, dp, vp], i),
        "sv_exchange_stage": ([vp, vp, i, i, ctypes.POINTER(SvGate), i, vp], i),
        "sv_norm_sq": ([vp, i, i, vp, vp], i),
        "sv_init_random": ([vp, i, u64, u64, vp], i),
        "sv_scale": ([vp, i, ctypes.c_double, vp], i),
        "sv_init_basis": ([vp, i, i64, vp], i),
        "sv_copy": ([vp, vp, u64, vp], i),
        "sv_ipc_handle": ([vp, vp, ctypes.POINTER(u64)], i),
        "sv_ipc_open": ([vp, u64, ctypes.POINTER(vp)], i),
        "sv_ipc_close": ([vp, u64], i),
        "sv_diag_global": ([vp, i, i, i, dp, vp, vp, vp], i),
        "sv_diag_fix": ([vp, i, i, i, dp, vp, vp, vp], i),
        "sv_swap_global": ([vp, vp, i, i, i, vp], i),
        "sv_max_abs_diff": ([vp, vp, i, vp, vp], i),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    if L.sv_version() != ABI_VERSION:
        raise ImportError(f"libsvb200 ABI {L.sv_version()} != expected {ABI_VERSION}; rebuild")
    _lib = L
    return L


def check(rc: int) -> None:
    if rc == SV_OK:
        return
    msg = (load().sv_last_error() or b"").decode(errors="replace")
    if rc == SV_EINVAL:
        raise ValueError(msg)
    raise NativeError(msg)


def qbuf(mat) -> ctypes.Array:
    """8 doubles q11re,q11im,q12re,q12im,q21re,q21im,q22re,q22im of a 2x2 complex matrix."""
    import numpy as np

    flat = np.ascontiguousarray(np.asarray(mat, dtype=np.complex128).reshape(4)).view(np.float64)
    return (ctypes.c_double * 8)(*flat.tolist())


def diag_sign_bytes(m: int) -> int:
    """SV_DIAG_SIGN_BYTES(m): sign map of sv_diag_global (2 bits per element, 8 bytes per 32)."""
    return ((1 << m) + 31) // 32 * 8


def launch_count() -> int:
    return int(load().sv_launch_count())
