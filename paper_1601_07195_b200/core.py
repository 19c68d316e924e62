"""Device-resident register (mirror of pkg/src/svsim/core.py).

A global n-qubit state of 2^n complex128 amplitudes is split over 2^p ranks
(one GPU each); rank r owns the contiguous slice of global indices
[r*2^m, (r+1)*2^m), m = n - p, so qubit k < m is bit k of the local index and
qubits m..n-1 are the rank bits (core.py:1-7).  The slice is one torch
complex128 CUDA tensor (interleaved re/im float64 = CUDA double2, allocated by
torch's caching allocator, 512-B aligned); torch is used for allocation and
streams only, every update is a libsvb200 kernel.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass, field
from typing import TYPE_CHECKING

import numpy as np
import torch

from . import _lib
from .errors import LayoutError
from .kernels import device_view, stream_handle

if TYPE_CHECKING:
    from .distributed import NvlinkFabric

AMP_BYTES = 16
ALIGNMENT = 64
_UIDS = itertools.count(1)


@dataclass(frozen=True)
class Layout:
    """Placement of one rank's slice: n qubits, 2^p ranks, this rank's id (core.py:27-64)."""

    n: int
    p: int = 0
    rank: int = 0

    def __post_init__(self):
        if self.n < 1:
            raise ValueError(f"need at least one qubit, got n={self.n}")
        if not 0 <= self.p < self.n:
            raise LayoutError(f"rank exponent p={self.p} must satisfy 0 <= p < n={self.n}")
        if not 0 <= self.rank < self.num_ranks:
            raise LayoutError(f"rank {self.rank} out of range for {self.num_ranks} ranks")

    @property
    def m(self) -> int:
        return self.n - self.p

    @property
    def num_ranks(self) -> int:
        return 1 << self.p

    @property
    def local_len(self) -> int:
        return 1 << self.m

    def global_index(self, local: int) -> int:
        return (self.rank << self.m) + local

    def split_global(self, g: int) -> tuple[int, int]:
        return g >> self.m, g & (self.local_len - 1)


def _device(device) -> torch.device:
    if device is None:
        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device: the B200 register has no host fallback")
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device)
    if d.type != "cuda":
        raise TypeError("the register lives in GPU memory; pass a CUDA device")
    if d.index is None:
        d = torch.device("cuda", torch.cuda.current_device())
    return d


def aligned_zeros(num_amps: int, device=None) -> torch.Tensor:
    """Zeroed complex128 device vector (core.py:67-75; torch blocks are 512-B aligned)."""
    return torch.zeros(num_amps, dtype=torch.complex128, device=_device(device))


@dataclass
class LocalState:
    """One rank's slice (device tensor) plus its layout; `corrupt` marks an aborted exchange."""

    layout: Layout
    amps: torch.Tensor
    corrupt: bool = field(default=False, compare=False)
    # process-unique id: peer mappings are keyed by it, so a new slice that happens to
    # reuse a freed slice's address never inherits that slice's stale mappings
    uid: int = field(default_factory=lambda: next(_UIDS), compare=False, repr=False)

    def __post_init__(self):
        if not isinstance(self.amps, torch.Tensor) or self.amps.dtype != torch.complex128:
            raise TypeError("amplitudes must be a complex128 torch tensor")
        if not self.amps.is_cuda:
            raise TypeError("amplitudes must live on a CUDA device")
        if tuple(self.amps.shape) != (self.layout.local_len,):
            raise LayoutError(
                f"slice length {tuple(self.amps.shape)} does not match 2^m = {self.layout.local_len}"
            )
        if not self.amps.is_contiguous():
            raise LayoutError("slice must be contiguous")

    @property
    def device(self) -> torch.device:
        return self.amps.device

    def copy(self) -> "LocalState":
        return LocalState(self.layout, self.amps.clone(), self.corrupt)

    def to_numpy(self) -> np.ndarray:
        return self.amps.cpu().numpy()

    def load_host(self, host: torch.Tensor) -> None:
        """Stream-ordered upload of this slice from a (pinned) host tensor via sv_copy."""
        self._host_copy(host, upload=True)

    def store_host(self, host: torch.Tensor) -> None:
        """Stream-ordered download of this slice into a (pinned) host tensor via sv_copy."""
        self._host_copy(host, upload=False)

    def _host_copy(self, host: torch.Tensor, upload: bool) -> None:
        if host.dtype != torch.complex128 or host.numel() != self.layout.local_len or not host.is_contiguous():
            raise LayoutError("host buffer must be a contiguous complex128 vector of 2^m elements")
        if host.is_cuda:
            raise TypeError("host buffer must live in host memory")
        dst, src = (self.amps.data_ptr(), host.data_ptr()) if upload else (host.data_ptr(), self.amps.data_ptr())
        with torch.cuda.device(self.amps.device):
            _lib.check(_lib.load().sv_copy(dst, src, self.layout.local_len * AMP_BYTES, stream_handle()))


def init_basis_state(layout: Layout, basis_index: int = 0, device=None) -> LocalState:
    """|basis_index>, sliced for this rank (core.py:104-112), written by sv_init_basis."""
    if not 0 <= basis_index < (1 << layout.n):
        raise ValueError(f"basis index {basis_index} out of range for n={layout.n}")
    dev = _device(device)
    amps = torch.empty(layout.local_len, dtype=torch.complex128, device=dev)
    owner, local = layout.split_global(basis_index)
    with torch.cuda.device(dev):
        _lib.check(_lib.load().sv_init_basis(amps.data_ptr(), layout.m, local if owner == layout.rank else -1,
                                             stream_handle()))
    return LocalState(layout, amps)


def state_from_global(layout: Layout, full, device=None) -> LocalState:
    """This rank's slice of a full 2^n host (or device) vector, uploaded (core.py:115-122)."""
    if tuple(full.shape) != (1 << layout.n,):
        raise LayoutError(f"full vector must have 2^n = {1 << layout.n} entries")
    dev = _device(device)
    start = layout.rank << layout.m
    part = full[start:start + layout.local_len]
    if isinstance(part, np.ndarray):
        part = torch.from_numpy(np.ascontiguousarray(part, dtype=np.complex128))
    amps = part.to(device=dev, dtype=torch.complex128, copy=True).contiguous()
    return LocalState(layout, amps)


def _partial_norm(state: LocalState, qubit: int) -> float:
    ptr, m = device_view(state.amps)
    scratch = torch.empty(_lib.SV_NORM_SCRATCH, dtype=torch.float64, device=state.amps.device)
    with torch.cuda.device(state.amps.device):
        _lib.check(_lib.load().sv_norm_sq(ptr, m, qubit, scratch.data_ptr(), stream_handle()))
    return float(scratch[-1].item())


def _reduce_sum(partial: float, layout: Layout, transport: "NvlinkFabric | None") -> float:
    """Rank-ordered sum of per-rank partials, same total on every rank (core.py:125-144)."""
    if layout.p == 0:
        return partial
    if transport is None:
        raise LayoutError("cross-rank reduction requires a transport when p > 0")
    return transport.reduce_sum(partial)


def max_abs_diff(a: torch.Tensor, b: torch.Tensor) -> float:
    """max |a_i - b_i| over two device slices of the same length (sv_max_abs_diff)."""
    pa, m = device_view(a)
    pb, mb = device_view(b)
    if m != mb:
        raise ValueError(f"slices differ in length: 2^{m} vs 2^{mb}")
    scratch = torch.empty(_lib.SV_NORM_SCRATCH, dtype=torch.float64, device=a.device)
    with torch.cuda.device(a.device):
        _lib.check(_lib.load().sv_max_abs_diff(pa, pb, m, scratch.data_ptr(), stream_handle()))
    return float(scratch[-1].item())


def global_norm_sq(state: LocalState, transport: "NvlinkFabric | None" = None) -> float:
    """Sum of |amplitude|^2 over the whole state (core.py:147-150)."""
    return _reduce_sum(_partial_norm(state, -1), state.layout, transport)


def probability_of_bit(state: LocalState, qubit: int, transport: "NvlinkFabric | None" = None) -> float:
    """Probability that `qubit` reads 1 (core.py:153-167)."""
    lay = state.layout
    if not 0 <= qubit < lay.n:
        raise ValueError(f"qubit {qubit} out of range for n={lay.n}")
    if qubit < lay.m:
        partial = _partial_norm(state, qubit)
    elif (lay.rank >> (qubit - lay.m)) & 1:
        partial = _partial_norm(state, -1)
    else:
        partial = 0.0
    return _reduce_sum(partial, lay, transport)


def init_random_state(layout: Layout, seed: int = 0, transport: "NvlinkFabric | None" = None,
                      device=None) -> LocalState:
    """Seeded i.i.d. complex Gaussian state normalised to unit global L2 norm, generated
    on the device (Philox counter = global index, so any sharding gives the same state).

    The BASELINE recipe (test_kernels.py:32-34) at sizes numpy cannot reach in
    reasonable time; for oracle parity use ``state_from_global`` on a numpy draw.
    """
    dev = _device(device)
    amps = torch.empty(layout.local_len, dtype=torch.complex128, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.load().sv_init_random(amps.data_ptr(), layout.m, int(seed) & (2**64 - 1),
                                              layout.rank, stream_handle()))
    st = LocalState(layout, amps)
    norm = global_norm_sq(st, transport) ** 0.5
    with torch.cuda.device(dev):
        _lib.check(_lib.load().sv_scale(amps.data_ptr(), layout.m, 1.0 / norm, stream_handle()))
    return st
