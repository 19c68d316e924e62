"""Gates on global qubits: pairwise NVLink exchange (mirror of pkg/src/svsim/distributed.py).

Rank r holds global indices [r*2^m, (r+1)*2^m).  A gate on qubit k >= m pairs
local element j of rank r with local element j of partner r ^ 2^(k-m)
(distributed.py:1-15).  The reference streams halves through a byte
transport in double-buffered chunks; here the data plane is the partner's
slice itself, mapped into this process with CUDA IPC, and the whole half
exchange is ONE kernel (``sv_exchange``): the zero side updates the first
half of every pair, the one side the second half, each reading the partner's
element over NVLink and storing the returned element straight back into the
partner's HBM.  Thousands of CTAs in flight overlap transfer and update, the
paper's T = max(T_comp, T_comm) pipeline (distributed.py:205-290) without
staging buffers or per-chunk host work.

Control plane (host): ``NvlinkFabric`` replaces the Transport ABC
(distributed.py:60-92).  It owns the process group, the IPC peer mappings,
the per-gate fences and the byte counters of ``CountingTransport``
(transport.py:549-598).  Fences are stream-ordered NCCL all-reduces of one
int (no host sync) when the group runs NCCL, host barriers otherwise.

Host logic is split from execution: ``plan_gate`` is the pure per-rank
decision of distributed.py:353-459 (which kernel, which partner, which half,
how many bytes), ``execute_action`` runs it against a device executor.
"""

from __future__ import annotations

import ctypes
import enum
import threading
import time
import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .core import AMP_BYTES, LocalState
from .errors import LayoutError, TransportError
from .kernels import (
    SERIAL,
    GateMatrix,
    ThreadPolicy,
    _as_gate,
    apply_controlled_raw,
    apply_single_raw,
    device_view,
    stream_handle,
)
from .perfmodel import BoundCase, classify_case

DEFAULT_CHUNK_BYTES = 4 << 20
GATHER_MAX_QUBITS = 26
CONTROL_TAG = 0


class ComputesHalf(enum.Enum):
    FIRST_HALF = 0
    SECOND_HALF = 1


@dataclass(frozen=True)
class ExchangePlan:
    """Who faces whom for one exchange, and the (API-compatible) chunking (distributed.py:100-122).

    The fused NVLink kernel has no staging buffers; chunk_amps / temp_capacity
    are validated exactly like the reference and otherwise only affect nothing:
    results are bitwise independent of them, as the reference guarantees.
    """

    partner: int
    this_rank_computes: ComputesHalf
    chunk_amps: int
    temp_capacity: int
    half_amps: int

    def __post_init__(self):
        if self.chunk_amps < 1:
            raise ValueError("chunk_amps must be >= 1")
        if self.half_amps % self.chunk_amps != 0:
            raise ValueError(f"chunk_amps {self.chunk_amps} must divide the half length {self.half_amps}")
        steps = self.half_amps // self.chunk_amps
        needed = self.chunk_amps * min(2, steps)
        if not needed <= self.temp_capacity <= self.half_amps:
            raise ValueError(f"temp_capacity {self.temp_capacity} outside [{needed}, {self.half_amps}]")


def make_exchange_plan(layout, k: int, *, chunk_amps: int | None = None, chunk_bytes: int | None = None,
                       temp_capacity: int | None = None) -> ExchangePlan:
    """Plan for pairing bit k >= m (distributed.py:125-158)."""
    m = layout.m
    if not m <= k < layout.n:
        raise LayoutError(f"qubit {k} is local (m={m}); no exchange needed")
    half = 1 << (m - 1)
    if chunk_amps is None:
        want = max(1, (chunk_bytes or DEFAULT_CHUNK_BYTES) // AMP_BYTES)
        chunk_amps = min(1 << (want.bit_length() - 1), half)
    steps = max(1, half // max(1, chunk_amps))
    if temp_capacity is None:
        temp_capacity = chunk_amps * min(2, steps)
    zero_side = ((layout.rank >> (k - m)) & 1) == 0
    return ExchangePlan(
        partner=layout.rank ^ (1 << (k - m)),
        this_rank_computes=ComputesHalf.FIRST_HALF if zero_side else ComputesHalf.SECOND_HALF,
        chunk_amps=chunk_amps,
        temp_capacity=temp_capacity,
        half_amps=half,
    )


class ScratchPool:
    """Recycled chunk buffers with high-water accounting (distributed.py:161-181).

    The fused IPC exchange stages nothing and never draws from it; the staged
    data planes (NCCL send/recv and copy-engine chunks) take their two chunk
    buffers here, so ``high_water_bytes`` is 2 * chunk * 16 B for them, the
    reference's bound.
    """

    def __init__(self):
        self._free: dict[int, list[torch.Tensor]] = {}
        self._lock = threading.Lock()
        self.outstanding_bytes = 0
        self.high_water_bytes = 0

    def take(self, num_amps: int, device=None) -> torch.Tensor:
        with self._lock:
            stack = self._free.get(num_amps)
            buf = stack.pop() if stack else torch.zeros(
                num_amps, dtype=torch.complex128,
                device=device if device is not None else torch.device("cuda", torch.cuda.current_device()))
            self.outstanding_bytes += num_amps * AMP_BYTES
            self.high_water_bytes = max(self.high_water_bytes, self.outstanding_bytes)
            return buf

    def give(self, buf: torch.Tensor) -> None:
        with self._lock:
            self._free.setdefault(buf.shape[0], []).append(buf)
            self.outstanding_bytes -= buf.shape[0] * AMP_BYTES


# ------------------------------------------------------------------ host logic


@dataclass(frozen=True)
class GateAction:
    """What one rank does for one gate (pure function of layout and gate)."""

    kind: str            # "single" | "controlled" | "exchange" | "diag" | "idle" (local no-op) | "idle_exchange"
    case: BoundCase
    target: int
    control: int | None
    partner: int = -1
    own_is_zero: bool = True
    c_local: int = -1    # >= 0: only local-bit-c elements cross (case 5)
    sent: int = 0        # payload bytes leaving this rank over NVLink
    received: int = 0

    @property
    def fenced(self) -> bool:
        """Every rank fences around cases 2/5/6 (participating or not)."""
        return self.kind in ("exchange", "diag", "idle_exchange")


def plan_gate(layout, target: int, control: int | None, diag: bool = False) -> GateAction:
    """Per-rank routing of distributed.py:314-459 (cases of perfmodel.py:30-38).

    diag=True (a diagonal gate under NvlinkFabric(diagonal_local=True)):
    the exchange of cases 2/5/6 becomes a local "diag" action that moves no payload."""
    m, rank = layout.m, layout.rank
    case = classify_case(target, control, m)
    action = _plan_gate(layout, target, control, m, rank, case)
    if diag and action.kind == "exchange":
        return GateAction("diag", case, action.target, action.control, partner=action.partner,
                          own_is_zero=action.own_is_zero, c_local=action.c_local)
    return action


def _plan_gate(layout, target, control, m, rank, case) -> GateAction:
    if control is None:
        if target < m:
            return GateAction("single", case, target, None)
        bit = target - m
        return GateAction("exchange", case, target, None, partner=rank ^ (1 << bit),
                          own_is_zero=((rank >> bit) & 1) == 0, sent=1 << (m + 4), received=1 << (m + 4))
    c, t = control, target
    if c < m and t < m:
        return GateAction("controlled", case, t, c)
    if t < m:  # case 4: control in the rank bits, target local
        on = (rank >> (c - m)) & 1
        return GateAction("single" if on else "idle", case, t, c)
    bit = t - m
    partner = rank ^ (1 << bit)
    zero = ((rank >> bit) & 1) == 0
    if c >= m:  # case 6: only control-set ranks exchange
        if (rank >> (c - m)) & 1:
            return GateAction("exchange", case, t, c, partner=partner, own_is_zero=zero,
                              sent=1 << (m + 4), received=1 << (m + 4))
        return GateAction("idle_exchange", case, t, c)
    # case 5: local control, remote target -- packed bit-c = 1 elements
    return GateAction("exchange", case, t, c, partner=partner, own_is_zero=zero, c_local=c,
                      sent=1 << (m + 3), received=1 << (m + 3))


# ------------------------------------------------------------ device executor


class CudaExecutor:
    """libsvb200 launches on the current stream (the only product executor)."""

    def single(self, state: LocalState, k: int, q: GateMatrix) -> None:
        apply_single_raw(state.amps, k, q)

    def controlled(self, state: LocalState, c: int, t: int, q: GateMatrix) -> None:
        apply_controlled_raw(state.amps, c, t, q)

    def exchange(self, state: LocalState, theirs: int, own_is_zero: bool, c_local: int, q: GateMatrix) -> None:
        ptr, m = device_view(state.amps)
        with torch.cuda.device(state.amps.device):
            _lib.check(_lib.load().sv_exchange(ptr, theirs, m, int(own_is_zero), int(c_local),
                                               _as_gate(q).qbuf(), stream_handle()))

    def exchange_chunk(self, state: LocalState, buf: torch.Tensor, own_is_zero: bool, c_local: int, q: GateMatrix,
                       j0: int, count: int) -> None:
        ptr, m = device_view(state.amps)
        with torch.cuda.device(state.amps.device):
            _lib.check(_lib.load().sv_exchange_chunk(ptr, buf.data_ptr(), m, int(own_is_zero), int(c_local),
                                                     _as_gate(q).qbuf(), j0, count, stream_handle()))

    def scratch(self, state: LocalState, num_amps: int) -> torch.Tensor:
        return torch.empty(num_amps, dtype=torch.complex128, device=state.amps.device)

    def view(self, state: LocalState, j0: int, num_amps: int) -> torch.Tensor:
        return state.amps[j0:j0 + num_amps]

    def pair_update(self, mine: torch.Tensor, buf: torch.Tensor, own_is_zero: bool, q: GateMatrix) -> None:
        """_pair_kernel on two contiguous chunk vectors (sv_pair_update)."""
        with torch.cuda.device(mine.device):
            _lib.check(_lib.load().sv_pair_update(mine.data_ptr(), buf.data_ptr(), mine.numel(), int(own_is_zero),
                                                  _as_gate(q).qbuf(), stream_handle()))

    def tensor(self, state: LocalState) -> torch.Tensor:
        return state.amps

    def buffer_device(self, state: LocalState) -> torch.device:
        return state.amps.device

    def ce_exchange(self, state: LocalState, theirs: int, own_is_zero: bool, segments, q: GateMatrix,
                    bufs) -> None:
        """Copy-engine data plane: for each (j0, count, c_local) segment of this rank's computing
        half, cudaMemcpyAsync the partner's elements into a local chunk buffer (copy-in stream),
        update with the exchange kernel (current stream), push the partner's results back
        (copy-out stream).  Two buffers: chunk i+1 streams in while chunk i computes and
        chunk i-1 drains."""
        ptr, m = device_view(state.amps)
        dev = state.amps.device
        lib = _lib.load()
        qb = _as_gate(q).qbuf()
        with torch.cuda.device(dev):
            main = torch.cuda.current_stream(dev)
            s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
            s_in.wait_stream(main)
            freed = [None] * len(bufs)  # event: buffer b's previous push-back is done
            for i, (j0, cnt, cl) in enumerate(segments):
                b = i % len(bufs)
                buf = bufs[b]
                if freed[b] is not None:
                    s_in.wait_event(freed[b])
                _lib.check(lib.sv_copy(buf.data_ptr(), theirs + j0 * AMP_BYTES, cnt * AMP_BYTES, s_in.cuda_stream))
                got = torch.cuda.Event()
                got.record(s_in)
                main.wait_event(got)
                _lib.check(lib.sv_exchange_chunk(ptr, buf.data_ptr(), m, int(own_is_zero), int(cl), qb, j0, cnt,
                                                 main.cuda_stream))
                done = torch.cuda.Event()
                done.record(main)
                s_out.wait_event(done)
                _lib.check(lib.sv_copy(theirs + j0 * AMP_BYTES, buf.data_ptr(), cnt * AMP_BYTES, s_out.cuda_stream))
                freed[b] = torch.cuda.Event()
                freed[b].record(s_out)
            main.wait_stream(s_out)
            main.wait_stream(s_in)

    def exchange_stage(self, state: LocalState, theirs: int, own_is_zero: bool, ops) -> None:
        from .kernels import gate_array

        ptr, m = device_view(state.amps)
        with torch.cuda.device(state.amps.device):
            _lib.check(_lib.load().sv_exchange_stage(ptr, theirs, m, int(own_is_zero), gate_array(ops), len(ops),
                                                     stream_handle()))

    def local_gates(self, state: LocalState, ops, tile: int = 0, group: int | None = None,
                    exact: bool = True) -> None:
        """sv_apply_gates_ex (planner inside), or sv_apply_group_ex for one pre-planned group;
        exact=False is the tolerance mode (SV_FLAG_TOLERANCE)."""
        from .kernels import apply_gates, gate_array

        if group is None:
            apply_gates(state.amps, ops, tile, exact=exact)
            return
        ptr, m = device_view(state.amps)
        with torch.cuda.device(state.amps.device):
            _lib.check(_lib.load().sv_apply_group_ex(ptr, m, int(group), gate_array(ops), len(ops), int(tile),
                                                     0 if exact else _lib.SV_FLAG_TOLERANCE, stream_handle()))

    def synchronize(self, state: LocalState) -> None:
        torch.cuda.current_stream(state.amps.device).synchronize()

    def key(self, state: LocalState) -> tuple:
        return (getattr(state, "uid", None), state.amps.data_ptr(), state.amps.numel(), str(state.amps.device))

    def flag_device(self, state: LocalState | None) -> torch.device:
        return state.amps.device if state is not None else torch.device("cuda", torch.cuda.current_device())

    def share(self, state: LocalState):
        """(64-byte IPC handle, byte offset) of the slice's allocation."""
        h = (ctypes.c_char * 64)()
        off = ctypes.c_uint64(0)
        with torch.cuda.device(state.amps.device):
            _lib.check(_lib.load().sv_ipc_handle(state.amps.data_ptr(), h, ctypes.byref(off)))
        return bytes(h), int(off.value)

    def open(self, state: LocalState, blob) -> int:
        handle, off = blob
        p = ctypes.c_void_p()
        with torch.cuda.device(state.amps.device):
            _lib.check(_lib.load().sv_ipc_open(ctypes.c_char_p(handle), off, ctypes.byref(p)))
        return int(p.value)

    def close(self, ptr: int, blob) -> None:
        _lib.check(_lib.load().sv_ipc_close(ptr, blob[1]))

    def copy(self, dst: int, src: int, nbytes: int, state: LocalState) -> None:
        with torch.cuda.device(state.amps.device):
            _lib.check(_lib.load().sv_copy(dst, src, nbytes, stream_handle()))

    def swap_global(self, state: LocalState, theirs: int, own_is_zero: bool, l: int) -> None:
        ptr, m = device_view(state.amps)
        with torch.cuda.device(state.amps.device):
            _lib.check(_lib.load().sv_swap_global(ptr, theirs, m, int(own_is_zero), int(l), stream_handle()))

    # --- diagonal global gates
    def diag_alloc(self, state: LocalState):
        """(sign map, flag) device buffers of sv_diag_global for this slice."""
        dev = state.amps.device
        return (torch.empty(_lib.diag_sign_bytes(state.layout.m), dtype=torch.uint8, device=dev),
                torch.zeros(1, dtype=torch.int32, device=dev))

    def share_buffer(self, state: LocalState, buf):
        h = (ctypes.c_char * 64)()
        off = ctypes.c_uint64(0)
        with torch.cuda.device(state.amps.device):
            _lib.check(_lib.load().sv_ipc_handle(buf.data_ptr(), h, ctypes.byref(off)))
        return bytes(h), int(off.value)

    def diag_global(self, state: LocalState, own_is_zero: bool, c_local: int, q: GateMatrix, signs, flag) -> None:
        ptr, m = device_view(state.amps)
        with torch.cuda.device(state.amps.device):
            _lib.check(_lib.load().sv_diag_global(ptr, m, int(own_is_zero), int(c_local), _as_gate(q).qbuf(),
                                                  signs.data_ptr(), flag.data_ptr(), stream_handle()))

    def diag_fix(self, state: LocalState, own_is_zero: bool, c_local: int, q: GateMatrix, peer_signs: int,
                 flag) -> None:
        ptr, m = device_view(state.amps)
        with torch.cuda.device(state.amps.device):
            _lib.check(_lib.load().sv_diag_fix(ptr, m, int(own_is_zero), int(c_local), _as_gate(q).qbuf(),
                                               peer_signs, flag.data_ptr(), stream_handle()))


_CUDA = CudaExecutor()


FP_MASK = (1 << 62) - 1


def fingerprint(*fields) -> int:
    """Deterministic 62-bit protocol word of one fenced step (same on every rank that agrees
    on the step; the reference's wire phase words, distributed.py:46-47)."""
    h = 0x345678
    for f in fields:
        h = ((h ^ (int(f) & 0xFFFFFFFFFFFF)) * 1000003 + 0x9E3779B1) & FP_MASK
    return h


class NvlinkFabric:
    """Exchange fabric over one torch.distributed group, one rank per GPU.

    Stands in for the reference's ``transport`` argument everywhere
    (apply_op, run_circuit, global_norm_sq, gather_full_state).  Counters
    follow CountingTransport: payload bytes sent / received over the link.

    Data planes: "ipc" (default, the product) -- the fused exchange kernel on
    the partner's CUDA-IPC-mapped slice; "ce" -- copy-engine chunks
    (cudaMemcpyAsync of peer chunks into a local double buffer, the exchange
    kernel, an async push back); "nccl" -- the reference's staged pipeline
    (distributed.py:205-290) over NCCL send/recv, double-buffered, at most two
    chunks in flight (the baseline, and the fallback when peer mapping is
    refused).

    Fences fail loudly (the reference's TransportError on a timeout or a phase
    desync, transport.py:56-79): every fence all-reduces (max) this rank's
    protocol fingerprint and its negation, so ranks that disagree on the step
    -- different gate, chunking or plan -- see max != min and raise
    ``TransportError``; a fence that does not complete within ``timeout_s``
    raises too.  Host fences (gloo) check at once; stream fences (NCCL) are
    checked without a host sync every ``check_every`` fences and at the end of
    each ``run_circuit`` (``check``).
    """

    def __init__(self, group=None, *, fence: str | None = None, executor=None, data_plane: str = "ipc",
                 chunk_amps: int = 1 << 26, diagonal_local: bool = False, timeout_s: float = 300.0,
                 check_every: int = 64):
        import torch.distributed as dist

        if not dist.is_initialized():
            raise TransportError("NvlinkFabric needs an initialised torch.distributed process group")
        self._dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.num_ranks = dist.get_world_size(group)
        backend = str(dist.get_backend(group)).lower()
        self.fence_mode = fence or ("stream" if backend == "nccl" else "host")
        if self.fence_mode not in ("stream", "host"):
            raise ValueError("fence must be 'stream' or 'host'")
        if data_plane not in ("ipc", "ce", "nccl"):
            raise ValueError("data_plane must be 'ipc', 'ce' or 'nccl'")
        self.data_plane = data_plane
        self.chunk_amps = chunk_amps
        self.scratch = ScratchPool()
        self.executor = executor or _CUDA
        self.sent_bytes = 0
        self.received_bytes = 0
        self.fences = 0
        self.timeout_s = float(timeout_s)
        self.check_every = int(check_every)
        self._pending: list = []
        self._tag = CONTROL_TAG
        self._lock = threading.Lock()
        self._peers: dict[tuple, tuple[list, list]] = {}
        # SURVEY.md 8(f)1, off by default (it departs from the reference's per-gate traffic
        # contract, test_acceptance.py:61-71): diagonal gates on global qubits run without an
        # exchange.  Must be the same on every rank.
        self.diagonal_local = bool(diagonal_local)
        self._diag: dict[tuple, tuple] = {}

    @property
    def diag_mode(self) -> bool:
        """Diagonal global gates take the no-exchange path (needs peer mappings)."""
        return self.diagonal_local and self.data_plane in ("ipc", "ce")

    @property
    def mapped(self) -> bool:
        """The data plane works on CUDA-IPC-mapped peer slices."""
        return self.data_plane in ("ipc", "ce")

    # --- Transport-compatible surface
    def fresh_tag(self) -> int:
        self._tag += 1
        return self._tag

    def snapshot(self) -> tuple[int, int]:
        with self._lock:
            return self.sent_bytes, self.received_bytes

    @property
    def total_bytes(self) -> int:
        return self.sent_bytes + self.received_bytes

    def count(self, sent: int, received: int) -> None:
        with self._lock:
            self.sent_bytes += sent
            self.received_bytes += received

    def exchange_objects(self, obj) -> list:
        out = [None] * self.num_ranks
        try:
            self._dist.all_gather_object(out, obj, group=self.group)
        except RuntimeError as exc:  # gloo/NCCL timeout or a dead peer
            raise TransportError(f"object exchange failed: {exc}") from exc
        return out

    def reduce_sum(self, partial: float) -> float:
        """Rank-ordered sum (deterministic, identical on every rank)."""
        total = 0.0
        for v in self.exchange_objects(float(partial)):
            total += v
        return total

    # --- fences
    def fence(self, state: LocalState | None = None, fp: int = 0) -> None:
        """Collective fence that also checks every rank is at the same protocol step."""
        import torch.distributed as dist

        self.fences += 1
        fp &= FP_MASK
        if self.fence_mode == "stream":
            dev = self.executor.flag_device(state)
            t = torch.empty(2, dtype=torch.int64, device=dev)
            t[0].fill_(fp)
            t[1].fill_(-fp)
            self._dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
            self._pending.append((fp, t, self.fences))
            if len(self._pending) >= self.check_every:
                self.check(state)
            return
        if state is not None:
            self.executor.synchronize(state)
        t = torch.tensor([fp, -fp], dtype=torch.int64)
        try:
            self._dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        except RuntimeError as exc:
            raise TransportError(f"fence {self.fences} failed or timed out: {exc}") from exc
        self._verify(fp, t, self.fences)

    def barrier(self, state: LocalState | None = None) -> None:
        """A fence with the neutral fingerprint (register/gather/teardown points)."""
        self.fence(state, 0)

    def _verify(self, fp: int, t, where: int) -> None:
        hi, lo = int(t[0]), -int(t[1])
        if hi != fp or lo != fp:
            raise TransportError(
                f"protocol desync at fence {where}: this rank is at step {fp:#x}, the ranks span "
                f"[{lo:#x}, {hi:#x}] (different gate, plan or chunking on some rank)")

    def check(self, state: LocalState | None = None) -> None:
        """Wait (at most timeout_s) for the stream fences issued so far and verify them."""
        if not self._pending:
            return
        pend, self._pending = self._pending, []
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(pend[-1][1].device))
        deadline = time.monotonic() + self.timeout_s
        while not ev.query():
            if time.monotonic() > deadline:
                raise TransportError(f"fence {pend[-1][2]} did not complete within {self.timeout_s:g} s "
                                     "(a rank diverged from the gate sequence or died)")
            time.sleep(2e-4)
        vals = torch.stack([t for _, t, _ in pend]).cpu()
        for (fp, _, where), v in zip(pend, vals):
            self._verify(fp, v, where)

    # --- peer mappings
    def ensure_registered(self, state: LocalState) -> None:
        """Collective: map every rank's slice into this process (once per slice).

        Every rank takes part in every collective whatever happens locally: the
        export blobs are all-gathered (None from a rank that failed), then every
        rank's success.  If any rank cannot export or map a slice, every rank
        drops its mappings and switches to the NCCL data plane together.  The
        sign maps of diagonal_local follow the same two-step pattern; if they
        fail anywhere, diagonal gates go back to exchanges on every rank."""
        if not self.mapped:
            return
        key = self.executor.key(state)
        if key in self._peers:
            return
        err = None
        mine = None
        try:
            mine = self.executor.share(state)
        except Exception as exc:  # noqa: BLE001 -- reported below, collectively
            err = exc
        blobs = self.exchange_objects(mine)
        ptrs = [None] * self.num_ranks
        if err is None and any(b is None for b in blobs):
            err = TransportError("a peer could not export its slice")
        if err is None:
            for r, blob in enumerate(blobs):
                if r == self.rank:
                    continue
                try:
                    ptrs[r] = self.executor.open(state, blob)
                except Exception as exc:  # noqa: BLE001
                    err = exc
                    break
        ok = self.exchange_objects(err is None)
        if not all(ok):
            self._close_all(ptrs, blobs)
            warnings.warn(f"peer mapping refused on some rank ({err!r} here); exchanges fall back to NCCL "
                          "send/recv")
            self.data_plane = "nccl"
            return
        self._peers[key] = (ptrs, blobs)
        if self.diagonal_local:
            self._register_signs(state, key)

    def _close_all(self, ptrs, blobs) -> None:
        for r, p in enumerate(ptrs):
            if p is not None:
                try:
                    self.executor.close(p, blobs[r])
                except Exception:  # noqa: BLE001 -- best effort while falling back
                    pass

    def _register_signs(self, state: LocalState, key) -> None:
        """Sign map + flag of this slice, and every peer's sign map mapped here (collective)."""
        err, blob, signs, flag = None, None, None, None
        try:
            signs, flag = self.executor.diag_alloc(state)
            blob = self.executor.share_buffer(state, signs)
        except Exception as exc:  # noqa: BLE001
            err = exc
        blobs = self.exchange_objects(blob)
        peers = [None] * self.num_ranks
        if err is None and any(b is None for b in blobs):
            err = TransportError("a peer could not export its sign map")
        if err is None:
            for r, b in enumerate(blobs):
                if r == self.rank:
                    continue
                try:
                    peers[r] = self.executor.open(state, b)
                except Exception as exc:  # noqa: BLE001
                    err = exc
                    break
        ok = self.exchange_objects(err is None)
        if all(ok):
            self._diag[key] = (signs, flag, peers, blobs)
            return
        self._close_all(peers, blobs)
        warnings.warn(f"sign-map registration failed on some rank ({err!r} here); diagonal global gates "
                      "exchange as usual")
        self.diagonal_local = False

    def diag_buffers(self, state: LocalState):
        try:
            signs, flag, _, _ = self._diag[self.executor.key(state)]
        except KeyError as exc:
            raise TransportError("slice not registered for diagonal global gates") from exc
        return signs, flag

    def peer_signs(self, state: LocalState, rank: int) -> int:
        try:
            return self._diag[self.executor.key(state)][2][rank]
        except (KeyError, IndexError) as exc:
            raise TransportError("peer sign map not registered") from exc

    # --- staged data planes
    def _global_peer(self, rank: int) -> int:
        return rank if self.group is None else self._dist.get_global_rank(self.group, rank)

    def staged_exchange(self, state: LocalState, action: GateAction, q: GateMatrix, chunk: int | None = None,
                        scratch: ScratchPool | None = None) -> int:
        """One gate's exchange on the staged planes ("nccl", "ce").  Returns the payload bytes
        this rank sent (== received)."""
        if self.data_plane == "ce":
            return ce_exchange(self, state, action, q, chunk, scratch)
        return self.nccl_exchange(state, action, q, chunk, scratch)

    def nccl_exchange(self, state: LocalState, action: GateAction, q: GateMatrix, chunk: int | None = None,
                      scratch: ScratchPool | None = None) -> int:
        """The reference's half exchange over send/recv (distributed.py:205-422): per half,
        the computing rank receives the partner's chunks into two scratch buffers, updates
        both with the pair kernel and returns the partner's elements; the passive rank streams
        its chunks out (at most two in flight) and receives them updated.  Case 5 packs the
        bit-c = 1 elements of each half first (``_packed_control_slice``), so only they cross."""
        ex = self.executor
        m = state.layout.m
        half = 1 << (m - 1)
        whole = ex.tensor(state)
        peer = self._global_peer(action.partner)
        pool = scratch if scratch is not None else self.scratch
        chunk = chunk or self.chunk_amps
        c = action.c_local
        moved = 0
        for stage in (0, 1):
            region = whole[stage * half:(stage + 1) * half]
            sel = None
            if c == m - 1:  # the half-selecting bit: only the second half holds control-set pairs
                if stage == 0:
                    continue
                vec = region
            elif c >= 0:
                sel = region.view(-1, 2, 1 << c)[:, 1, :]
                if sel.is_contiguous():  # c = m - 2: one run, already packed
                    vec, sel = sel.reshape(-1), None
                else:
                    vec = sel.contiguous().view(-1)
            else:
                vec = region
            computing = action.own_is_zero == (stage == 0)
            self._pipeline(state, vec, computing, action.own_is_zero, q, chunk, pool, peer)
            if sel is not None:
                sel.copy_(vec.view(sel.shape))
            moved += vec.numel() * AMP_BYTES
        return moved

    def _pipeline(self, state, vec, computing: bool, own_is_zero: bool, q, chunk: int, pool, peer: int) -> None:
        """chunked_exchange_pipeline (distributed.py:205-290) over torch.distributed p2p.
        Both sides issue their operations in one global order (computing: R0 R1 S0 R2 S1 R3 ...,
        passive: S0 S1 R0 S2 R1 S3 ...), so blocking (gloo) and stream-ordered (NCCL)
        transports pair them identically and never deadlock; NCCL overlaps chunk i+1's
        transfer with chunk i's update."""
        total = vec.numel()
        if total == 0:
            return
        chunk = min(chunk, total)
        steps = -(-total // chunk)
        span = [(i * chunk, min(total, (i + 1) * chunk)) for i in range(steps)]
        works = []
        if not computing:
            for i in range(min(2, steps)):
                works.append(self._isend(vec[span[i][0]:span[i][1]], peer))
            for i in range(steps):
                lo, hi = span[i]
                works.append(self._irecv(vec[lo:hi], peer))
                if i + 2 < steps:
                    works.append(self._isend(vec[span[i + 2][0]:span[i + 2][1]], peer))
            self._wait_all(works)
            return
        nbuf = min(2, steps)
        dev = self.executor.buffer_device(state)
        bufs = [pool.take(chunk, device=dev) for _ in range(nbuf)]
        try:
            recvs = {}
            for i in range(nbuf):
                lo, hi = span[i]
                recvs[i] = self._irecv(bufs[i % nbuf][:hi - lo], peer)
            for i in range(steps):
                lo, hi = span[i]
                buf = bufs[i % nbuf][:hi - lo]
                self._wait_all([recvs.pop(i)])
                self.executor.pair_update(vec[lo:hi], buf, own_is_zero, q)
                works.append(self._isend(buf, peer))
                if i + 2 < steps:
                    lo2, hi2 = span[i + 2]
                    recvs[i + 2] = self._irecv(bufs[i % nbuf][:hi2 - lo2], peer)
            self._wait_all(works)
        finally:
            for b in bufs:
                pool.give(b)

    def _isend(self, t: torch.Tensor, peer: int):
        if self.fence_mode == "host":  # gloo: blocking, host memory
            self._send(t, peer)
            return None
        return self._dist.isend(t, dst=peer, group=self.group)

    def _irecv(self, t: torch.Tensor, peer: int):
        if self.fence_mode == "host":
            self._recv(t, peer)
            return None
        return self._dist.irecv(t, src=peer, group=self.group)

    def _wait_all(self, works: list) -> None:
        for w in works:
            if w is not None:
                w.wait()  # NCCL: the current stream waits, the host does not
        works.clear()

    def _send(self, t: torch.Tensor, peer: int) -> None:
        if t.is_cuda and self.fence_mode == "host":  # gloo moves host memory only
            t = t.cpu()
        self._dist.send(t.contiguous(), dst=peer, group=self.group)

    def _recv(self, t: torch.Tensor, peer: int) -> None:
        if t.is_cuda and self.fence_mode == "host":
            tmp = torch.empty(t.shape, dtype=t.dtype)
            self._dist.recv(tmp, src=peer, group=self.group)
            t.copy_(tmp)
            return
        self._dist.recv(t, src=peer, group=self.group)

    def peer_pointer(self, state: LocalState, rank: int) -> int:
        key = self.executor.key(state)
        try:
            ptr = self._peers[key][0][rank]
        except KeyError as exc:
            raise TransportError("slice not registered with the fabric") from exc
        if ptr is None:
            raise TransportError(f"rank {rank} is this rank; no peer mapping")
        return ptr

    def release(self, state: LocalState) -> None:
        """Unmap the peers' slices registered for `state` (collective-free)."""
        key = self.executor.key(state)
        entry = self._peers.pop(key, None)
        if entry:
            self._close_all(*entry)
        diag = self._diag.pop(key, None)
        if diag:
            self._close_all(diag[2], diag[3])

    def close(self) -> None:
        for key in list(self._diag):
            _, _, ptrs, blobs = self._diag.pop(key)
            self._close_all(ptrs, blobs)
        for key in list(self._peers):
            ptrs, blobs = self._peers.pop(key)
            self._close_all(ptrs, blobs)


def ce_exchange(fabric, state: LocalState, action: GateAction, q: GateMatrix, chunk: int | None = None,
            scratch: ScratchPool | None = None) -> int:
    """Copy-engine data plane: this rank computes its half of the pair space (zero side the
    first, one side the second, as the fused kernel) through two local chunk buffers;
    chunks whose elements all have control bit c clear are skipped."""
    m = state.layout.m
    half = 1 << (m - 1)
    lo = 0 if action.own_is_zero else half
    c = action.c_local
    if c == m - 1:
        if action.own_is_zero:
            return 0
        c = -1
    chunk = min(chunk or fabric.chunk_amps, half)
    segs = []
    for j0 in range(lo, lo + half, chunk):
        if c >= 0 and (2 << c) > chunk:  # the chunk lies on one side of bit c
            if (j0 >> c) & 1:
                segs.append((j0, chunk, -1))
        else:
            segs.append((j0, chunk, c))
    pool = scratch if scratch is not None else fabric.scratch
    dev = fabric.executor.buffer_device(state)
    bufs = [pool.take(chunk, device=dev) for _ in range(min(2, len(segs)))]
    try:
        if segs:
            fabric.executor.ce_exchange(state, fabric.peer_pointer(state, action.partner), action.own_is_zero, segs,
                                      q, bufs)
    finally:
        for b in bufs:
            pool.give(b)
    return sum(cnt for _, cnt, _ in segs) * AMP_BYTES


class InprocFabric:
    """Every rank of a layout in ONE process on one device -- the reference's inproc
    transport (transport.py, driven by cli.py:266-288) without threads.  Rank r's slice is
    ``states[r]``; a peer mapping is the plain device pointer of the partner's slice, and
    the caller runs each gate rank by rank on one stream (engine.run_circuit_inproc), so
    stream order is the fence.  Same exchange kernels, same counters as NvlinkFabric."""

    diagonal_local = False
    diag_mode = False
    mapped = True

    def __init__(self, states, rank: int, data_plane: str = "ipc", chunk_amps: int = 1 << 26):
        if data_plane not in ("ipc", "ce"):
            raise ValueError("in-process ranks run the 'ipc' (fused kernel) or 'ce' (copy-engine) plane")
        self.states, self.rank, self.num_ranks = states, rank, len(states)
        self.data_plane = data_plane
        self.chunk_amps = chunk_amps
        self.scratch = ScratchPool()
        self.executor = _CUDA
        self.sent_bytes = self.received_bytes = 0
        self.fences = 0
        self._tag = CONTROL_TAG

    @classmethod
    def group(cls, states, data_plane: str = "ipc", chunk_amps: int = 1 << 26) -> list["InprocFabric"]:
        return [cls(states, r, data_plane, chunk_amps) for r in range(len(states))]

    def staged_exchange(self, state, action, q, chunk=None, scratch=None) -> int:
        return ce_exchange(self, state, action, q, chunk, scratch)

    def fence(self, state=None, fp: int = 0) -> None:
        self.fences += 1

    def check(self, state=None) -> None:
        pass

    def fresh_tag(self) -> int:
        self._tag += 1
        return self._tag

    def snapshot(self) -> tuple[int, int]:
        return self.sent_bytes, self.received_bytes

    @property
    def total_bytes(self) -> int:
        return self.sent_bytes + self.received_bytes

    def count(self, sent: int, received: int) -> None:
        self.sent_bytes += sent
        self.received_bytes += received

    def barrier(self, state=None) -> None:
        self.fences += 1

    def ensure_registered(self, state) -> None:
        pass

    def peer_pointer(self, state, rank: int) -> int:
        if rank == self.rank:
            raise TransportError(f"rank {rank} is this rank; no peer mapping")
        return self.states[rank].amps.data_ptr()

    def release(self, state) -> None:
        pass

    def close(self) -> None:
        pass


def _fence(fabric, state, fp: int) -> None:
    fence = getattr(fabric, "fence", None)
    if fence is not None:
        fence(state, fp)
    else:
        fabric.barrier(state)


def step_fingerprint(tag: int, target: int, control: int | None, chunk: int | None = None, what: int = 0) -> int:
    """Protocol word of one fenced gate: every participating and idle rank computes the same
    value when they agree on the gate, its plan's chunking and the step kind."""
    return fingerprint(tag, target, -1 if control is None else control, chunk or 0, what)


def execute_action(state: LocalState, action: GateAction, q: GateMatrix, fabric: NvlinkFabric | None,
                   executor=None, *, tag: int | None = None, chunk: int | None = None,
                   scratch: ScratchPool | None = None) -> None:
    """Run one rank's share of one gate; fences bracket every exchange-class gate on all ranks.
    A fence that finds the ranks at different steps, or times out, raises TransportError
    and marks the slice corrupt (distributed.py:293-311, transport.py:56-79)."""
    ex = executor or (fabric.executor if fabric is not None else _CUDA)
    if action.kind == "single":
        ex.single(state, action.target, q)
    elif action.kind == "controlled":
        ex.controlled(state, action.control, action.target, q)
    if not action.fenced:
        return
    if fabric is None:
        raise LayoutError(f"gate on qubit {action.target} needs a transport")
    # rank-independent: participating, idle and diagonal-path ranks all fence with the same word
    fp = step_fingerprint(getattr(fabric, "_tag", 0) if tag is None else tag, action.target, action.control, chunk)
    if action.kind == "diag":
        _execute_diag(state, action, q, fabric, ex, fp)
        return
    try:
        # Partner slices are read and written in place: every rank's prior
        # work must be complete before, and the exchange complete after.
        _fence(fabric, state, fp)
        plane = getattr(fabric, "data_plane", "ipc")
        if action.kind == "exchange" and plane in ("nccl", "ce"):
            moved = fabric.staged_exchange(state, action, q, chunk, scratch)
            fabric.count(moved, moved)
        else:
            if action.kind == "exchange":
                ex.exchange(state, fabric.peer_pointer(state, action.partner), action.own_is_zero, action.c_local,
                            q)
            fabric.count(action.sent, action.received)
        _fence(fabric, state, fp)
    except TransportError:
        state.corrupt = True
        raise
    except Exception as exc:  # a failed collective (timeout, dead peer) surfaces as the reference's error
        state.corrupt = True
        if isinstance(exc, (ValueError, LayoutError)):
            raise
        raise TransportError(f"exchange for qubit {action.target} failed: {exc}") from exc
    except BaseException:
        state.corrupt = True
        raise


def _execute_diag(state, action, q, fabric, ex, fp: int = 0) -> None:
    """Diagonal gate on a global qubit without an exchange (sv_diag_global / sv_diag_fix):
    own elements multiplied in place, then -- after a fence, so the partner's sign map of
    its original elements is complete -- zero components patched from that map.  The
    trailing fence keeps the next diagonal gate from overwriting a map the partner still
    reads.  Idle ranks (case 6, control bit clear) take two fences either way."""
    try:
        signs, flag = fabric.diag_buffers(state)
        ex.diag_global(state, action.own_is_zero, action.c_local, q, signs, flag)
        _fence(fabric, state, fp)
        ex.diag_fix(state, action.own_is_zero, action.c_local, q, fabric.peer_signs(state, action.partner), flag)
        fabric.count(0, 0)
        _fence(fabric, state, fp)
    except BaseException:
        state.corrupt = True
        raise


def is_diagonal(q) -> bool:
    """q12 == q21 == 0 exactly (either zero sign): the diagonal fast path applies."""
    mat = _as_gate(q).mat
    return mat[0, 1] == 0 and mat[1, 0] == 0


# ------------------------------------------------------------- reference API


def _check_transport(transport, lay):
    if transport is None:
        raise LayoutError("distributed gate application needs a transport")
    if transport.num_ranks != lay.num_ranks or transport.rank != lay.rank:
        raise LayoutError(
            f"fabric rank {transport.rank}/{transport.num_ranks} does not match layout "
            f"rank {lay.rank}/{lay.num_ranks}")


def apply_single_distributed(state: LocalState, k: int, q: GateMatrix, transport: NvlinkFabric, *,
                             plan: ExchangePlan | None = None, chunk_amps: int | None = None,
                             scratch: ScratchPool | None = None, policy: ThreadPolicy = SERIAL) -> None:
    """Single-qubit gate on global qubit k >= m via the fused half exchange (distributed.py:314-338)."""
    lay = state.layout
    if lay.p < 1:
        raise LayoutError("distributed gate application needs at least 2 ranks")
    if not lay.m <= k < lay.n:
        raise LayoutError(f"qubit {k} is local (m={lay.m}); use the local kernel")
    explicit = plan.chunk_amps if plan is not None else chunk_amps
    if plan is None:
        plan = make_exchange_plan(lay, k, chunk_amps=chunk_amps)
    apply_global(state, k, None, q, transport, plan=plan, chunk=explicit, scratch=scratch)


def apply_controlled_distributed(state: LocalState, c: int, t: int, q: GateMatrix, transport: NvlinkFabric, *,
                                 plan: ExchangePlan | None = None, chunk_amps: int | None = None,
                                 scratch: ScratchPool | None = None, policy: ThreadPolicy = SERIAL) -> None:
    """Controlled gate with a qubit in the rank bits: cases 4, 5, 6 (distributed.py:353-422)."""
    lay = state.layout
    if c == t:
        raise ValueError(f"control and target must differ, both are {c}")
    if not (0 <= c < lay.n and 0 <= t < lay.n):
        raise ValueError(f"qubits ({c},{t}) out of range for n={lay.n}")
    if lay.p < 1:
        raise LayoutError("distributed gate application needs at least 2 ranks")
    m = lay.m
    if c < m and t < m:
        apply_controlled_raw(state.amps, c, t, q, policy)
        return
    explicit = plan.chunk_amps if plan is not None else chunk_amps
    if t >= m and plan is None:
        plan = make_exchange_plan(lay, t, chunk_amps=chunk_amps)
    apply_global(state, t, c, q, transport, plan=plan, chunk=explicit, scratch=scratch)


def apply_global(state, target: int, control: int | None, q, transport, *, plan: ExchangePlan | None = None,
                 executor=None, chunk: int | None = None, scratch: ScratchPool | None = None) -> None:
    """Shared tail of the distributed entry points: one gate touching a rank bit.

    Every rank calls it for every such gate (SPMD), so the collective pieces
    -- fresh tag, slice registration, fences -- line up across ranks.  ``chunk``
    (the caller's explicit plan / chunk_amps) sets the staged planes' chunking
    and enters the fence fingerprint, so ranks with different plans fail loudly
    (the reference's test_mismatched_plans_fail_loudly, pkg/tests/test_distributed.py:218-235).
    """
    lay = state.layout
    _check_transport(transport, lay)
    tag = transport.fresh_tag()
    transport.ensure_registered(state)  # collective; may switch every rank to the NCCL data plane
    diag = getattr(transport, "diag_mode", False) and is_diagonal(q)
    action = plan_gate(lay, target, control, diag=diag)
    if plan is not None and action.kind == "exchange" and (
            plan.partner != action.partner
            or (plan.this_rank_computes is ComputesHalf.FIRST_HALF) != action.own_is_zero):
        state.corrupt = True
        raise TransportError("exchange plan does not match this rank's pairing")
    execute_action(state, action, _as_gate(q), transport, executor, tag=tag, chunk=chunk, scratch=scratch)


def apply_op(state: LocalState, op, transport: NvlinkFabric | None = None, *, policy: ThreadPolicy = SERIAL,
             chunk_amps: int | None = None, scratch: ScratchPool | None = None) -> None:
    """Route one GateOp to the local kernel or the exchange (distributed.py:425-459)."""
    from .kernels import apply_controlled_local, apply_single_local

    m = state.layout.m
    if op.control is None:
        if op.target < m:
            apply_single_local(state, op.target, op.gate, policy)
            return
        if transport is None:
            raise LayoutError(f"gate on qubit {op.target} >= m={m} requires a transport")
        apply_single_distributed(state, op.target, op.gate, transport, chunk_amps=chunk_amps, scratch=scratch,
                                 policy=policy)
        return
    if op.control < m and op.target < m:
        apply_controlled_local(state, op.control, op.target, op.gate, policy)
        return
    if transport is None:
        raise LayoutError(f"gate on qubits ({op.control},{op.target}) crosses m={m}; requires a transport")
    apply_controlled_distributed(state, op.control, op.target, op.gate, transport, chunk_amps=chunk_amps,
                                 scratch=scratch, policy=policy)


def gather_full_state(state: LocalState, transport: NvlinkFabric | None = None,
                      cap: int = GATHER_MAX_QUBITS) -> np.ndarray | None:
    """Rank-ordered concatenation on rank 0 (None elsewhere), read over NVLink (distributed.py:462-482)."""
    lay = state.layout
    if lay.n > cap:
        raise LayoutError(f"gather of 2^{lay.n} amplitudes exceeds the n <= {cap} guard")
    if lay.p == 0:
        return state.to_numpy()
    if transport is None:
        raise LayoutError("gather requires a transport when p > 0")
    _check_transport(transport, lay)
    tag = transport.fresh_tag()
    transport.ensure_registered(state)
    _fence(transport, state, fingerprint(tag, 0x6A7E))
    full = None
    nccl = getattr(transport, "data_plane", "ipc") == "nccl"
    if lay.rank == 0:
        dev = torch.empty(1 << lay.n, dtype=torch.complex128, device=state.amps.device)
        nbytes = lay.local_len * AMP_BYTES
        dev[: lay.local_len].copy_(state.amps)
        for src in range(1, lay.num_ranks):
            if nccl:
                transport._recv(dev[src << lay.m:(src + 1) << lay.m], src)
            else:
                transport.executor.copy(dev[src << lay.m:].data_ptr(), transport.peer_pointer(state, src), nbytes,
                                        state)
        full = dev.cpu().numpy()
    elif nccl:
        transport._send(state.amps, 0)
    _fence(transport, state, fingerprint(tag, 0x6A7E))
    check = getattr(transport, "check", None)
    if check is not None:
        check(state)
    return full
