"""Multi-rank host protocol on CPU: world_size 2/4/8 processes over gloo.

The product's control plane runs for real -- NvlinkFabric (object all-gather
for slice registration, host fences, byte counters, tags), plan_gate,
apply_global and execute_action -- with the device swapped for a test
executor: slices live in POSIX shared memory (standing in for IPC-mapped
HBM) and the kernels are the oracle's C restatement (standing in for
libsvb200).  The gathered state and every per-gate, per-rank byte count must
equal what the reference itself produced (tests/golden/circuits_small.npz).
"""

from __future__ import annotations

import ctypes
import os
import socket
import tempfile
from dataclasses import dataclass, field
from multiprocessing import shared_memory

import numpy as np
import pytest

from conftest import unpack_ops


@dataclass
class ShmState:
    layout: object
    amps: np.ndarray
    shm: object
    corrupt: bool = field(default=False)


class ShmOracleExecutor:
    """Test double of CudaExecutor: shm 'peer mappings', oracle 'kernels'."""

    def __init__(self):
        self._open = {}

    def single(self, state, k, q):
        from oracle import oracle

        oracle.apply_single(state.amps, k, q.mat)

    def controlled(self, state, c, t, q):
        from oracle import oracle

        oracle.apply_controlled(state.amps, c, t, q.mat)

    def exchange(self, state, theirs, own_is_zero, c_local, q):
        from oracle import oracle

        oracle.exchange_raw(state.amps.ctypes.data, theirs, state.layout.m, own_is_zero, c_local, q.mat)

    def exchange_chunk(self, state, buf, own_is_zero, c_local, q, j0, count):
        from oracle import oracle

        oracle.exchange_chunk_raw(state.amps.ctypes.data, buf.data_ptr(), state.layout.m, own_is_zero, c_local,
                                  q.mat, j0, count)

    def pair_update(self, mine, buf, own_is_zero, q):
        from oracle import oracle

        oracle.exchange_chunk_raw(mine.data_ptr(), buf.data_ptr(), 0, own_is_zero, -1, q.mat, 0, mine.numel())

    def tensor(self, state):
        import torch

        return torch.from_numpy(state.amps)

    def buffer_device(self, state):
        import torch

        return torch.device("cpu")

    def ce_exchange(self, state, theirs, own_is_zero, segments, q, bufs):
        """Copy-engine plane stand-in: partner chunk -> local buffer -> pair update -> back."""
        from oracle import oracle

        m = state.layout.m
        w = np.frombuffer((ctypes.c_char * (16 << m)).from_address(theirs), dtype=np.complex128)
        for i, (j0, cnt, cl) in enumerate(segments):
            buf = bufs[i % len(bufs)][:cnt]
            buf.numpy()[:] = w[j0:j0 + cnt]
            oracle.exchange_chunk_raw(state.amps.ctypes.data, buf.data_ptr(), m, own_is_zero, cl, q.mat, j0, cnt)
            w[j0:j0 + cnt] = buf.numpy()

    def scratch(self, state, num_amps):
        import torch

        return torch.empty(num_amps, dtype=torch.complex128)

    def view(self, state, j0, num_amps):
        import torch

        return torch.from_numpy(state.amps[j0:j0 + num_amps])

    def exchange_stage(self, state, theirs, own_is_zero, ops):
        # a same-target stage == its gates' exchanges in order (each keeps the half split)
        for op in ops:
            self.exchange(state, theirs, own_is_zero, -1 if op.control is None else op.control, op.gate)

    def local_gates(self, state, ops, tile=0, group=None):
        from oracle import oracle

        for op in ops:
            oracle.apply_gate(state.amps, (op.target, op.control, op.gate.mat))

    def synchronize(self, state):
        pass

    # diagonal global gates: the "sign map" stand-in is a shm snapshot of the original slice;
    # diag_fix forms the reference's mix() from it (the protocol under test: registration,
    # fences, partner map reads -- the split arithmetic itself is covered on the GPU)
    def diag_alloc(self, state):
        shm = shared_memory.SharedMemory(create=True, size=16 << state.layout.m,
                                         name=f"svd_{os.getpid()}_{state.layout.rank}")
        self._own = getattr(self, "_own", []) + [shm]
        return ShmState(state.layout, np.ndarray((1 << state.layout.m,), dtype=np.complex128, buffer=shm.buf),
                        shm), None

    def share_buffer(self, state, buf):
        return (buf.shm.name, 0)

    def diag_global(self, state, own_is_zero, c_local, q, signs, flag):
        signs.amps[:] = state.amps

    def diag_fix(self, state, own_is_zero, c_local, q, peer, flag):
        m = state.layout.m
        w = np.frombuffer((ctypes.c_char * (16 << m)).from_address(peer), dtype=np.complex128)
        x = state.amps
        sel = slice(None) if c_local < 0 else ((np.arange(1 << m) >> c_local) & 1).astype(bool)
        mat = q.mat
        if own_is_zero:
            out = mat[0, 0] * x[sel]
            out += mat[0, 1] * w[sel]
        else:
            out = mat[1, 0] * w[sel]
            out += mat[1, 1] * x[sel]
        x[sel] = out

    def swap_global(self, state, theirs, own_is_zero, l):
        m = state.layout.m
        w = np.frombuffer((ctypes.c_char * (16 << m)).from_address(theirs), dtype=np.complex128)
        quarter = 1 << (m - 2)
        j = np.arange(quarter, dtype=np.int64) + (0 if own_is_zero else quarter)
        z = ((j >> l) << (l + 1)) | (j & ((1 << l) - 1))
        im, it = (z | (1 << l), z) if own_is_zero else (z, z | (1 << l))
        x = state.amps[im].copy()
        state.amps[im] = w[it]
        w[it] = x

    def cleanup(self):
        for shm in getattr(self, "_own", []):
            shm.close()
            shm.unlink()

    def key(self, state):
        return state.shm.name

    def flag_device(self, state):
        raise AssertionError("host fences only")

    def share(self, state):
        return (state.shm.name, 0)

    def open(self, state, blob):
        shm = shared_memory.SharedMemory(name=blob[0])
        self._open[blob[0]] = shm
        return ctypes.addressof(ctypes.c_char.from_buffer(shm.buf)) + blob[1]

    def close(self, ptr, blob):
        shm = self._open.pop(blob[0], None)
        if shm is not None:
            try:
                shm.close()
            except BufferError:  # ctypes view still alive; unmapped at exit
                pass


def _worker(rank, world, port, path, name, n, plane="ipc"):
    import torch.distributed as dist

    import paper_1601_07195_b200 as sv

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        p = world.bit_length() - 1
        d = dict(np.load(path + ".npz"))
        lay = sv.Layout(n, p, rank)
        m = lay.m
        shm = shared_memory.SharedMemory(create=True, size=16 << m, name=f"svt_{os.getpid()}_{rank}")
        amps = np.ndarray((1 << m,), dtype=np.complex128, buffer=shm.buf)
        amps[:] = d["init"][rank << m:(rank + 1) << m]
        state = ShmState(lay, amps, shm)
        ex = ShmOracleExecutor()
        fabric = sv.NvlinkFabric(fence="host", executor=ex, data_plane=plane, chunk_amps=1 << max(0, m - 3))
        if plane != "ipc":  # the gather below maps the peers' shared memory
            fabric.data_plane = "ipc"
            fabric.ensure_registered(state)
            fabric.data_plane = plane
        deltas = []
        for t, c, q in zip(d["t"], d["c"], d["q"]):
            t, c, gate = int(t), None if c < 0 else int(c), sv.GateMatrix.unchecked(q.reshape(2, 2))
            before = fabric.snapshot()
            if max(t, -1 if c is None else c) < m:
                (ex.single(state, t, gate) if c is None else ex.controlled(state, c, t, gate))
            else:
                sv.apply_global(state, t, c, gate, fabric)
            after = fabric.snapshot()
            deltas.append((after[0] - before[0], after[1] - before[1]))
        total = fabric.reduce_sum(float(np.sum(np.abs(amps) ** 2)))
        blobs = fabric.exchange_objects(np.asarray(deltas, dtype=np.int64))
        fabric.barrier()
        if rank == 0:
            full = np.concatenate([amps.copy()] + [
                np.ndarray((1 << m,), dtype=np.complex128, buffer=ex._open[f"svt_{pid}_{r}"].buf).copy()
                for r, pid in enumerate(fabric.exchange_objects(os.getpid())) if r != 0])
        else:
            fabric.exchange_objects(os.getpid())
        fabric.barrier()
        if rank == 0:
            np.savez(path + ".out.npz", full=full, deltas=np.stack(blobs), norm=total, tags=fabric._tag,
                     fences=fabric.fences)
        fabric.barrier()
        fabric.close()
        del amps
        shm.close()
        shm.unlink()
    finally:
        dist.destroy_process_group()


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def run_world(world, name, n, golden, plane="ipc"):
    import torch.multiprocessing as mp

    d = golden("circuits_small")
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "w")
        np.savez(path + ".npz", init=d[f"{name}_in"], t=d[f"{name}_t"], c=d[f"{name}_c"], q=d[f"{name}_q"])
        mp.spawn(_worker, args=(world, _port(), path, name, n, plane), nprocs=world, join=True)
        return dict(np.load(path + ".out.npz")), d


@pytest.mark.parametrize("world,name,n", [(2, "mix10", 10), (4, "ctl12", 12), (2, "ctl12", 12)])
def test_gloo_nccl_data_plane_matches_reference(golden, world, name, n):
    """The staged send/recv data plane (baseline / fallback) gives the same bits and, with case 5
    packed to the bit-c = 1 elements, the reference's own per-gate byte counts -- with chunks
    smaller than 2^(c+1) for the high controls (chunk = 2^(m-3))."""
    out, d = run_world(world, name, n, golden, plane="nccl")
    p = world.bit_length() - 1
    assert np.array_equal(out["full"], d[f"{name}_p{p}"])
    assert np.array_equal(out["deltas"], d[f"{name}_p{p}_bytes"])


@pytest.mark.parametrize("world,name,n", [(2, "mix10", 10), (4, "ctl12", 12)])
def test_gloo_ce_data_plane_matches_reference(golden, world, name, n):
    """The copy-engine plane's chunk segmentation (skipping chunks on the clear side of a high
    control bit) gives the same bits as the reference."""
    out, d = run_world(world, name, n, golden, plane="ce")
    p = world.bit_length() - 1
    assert np.array_equal(out["full"], d[f"{name}_p{p}"])


@pytest.mark.parametrize("world,name,n", [(2, "mix10", 10), (4, "mix8", 8), (8, "ctl12", 12)])
def test_gloo_world_matches_reference(golden, world, name, n):
    out, d = run_world(world, name, n, golden)
    p = world.bit_length() - 1
    assert np.array_equal(out["full"], d[f"{name}_p{p}"])
    assert np.array_equal(out["deltas"], d[f"{name}_p{p}_bytes"])
    assert abs(float(out["norm"]) - 1.0) < 1e-12
    m = n - p
    glob = sum(1 for t, c, _ in unpack_ops(d, name) if max(t, -1 if c is None else c) >= m)
    assert int(out["tags"]) == glob            # one fresh tag per global-qubit gate, on every rank
    fenced = sum(1 for t, c, _ in unpack_ops(d, name) if t >= m)
    assert int(out["fences"]) == 2 * fenced + 2  # two fences per exchange-class gate + two final barriers


def _worker_passes(rank, world, port, path, n):
    """Pass-fused execution (FusionConfig(passes=True) semantics): global stages exchange once."""
    import torch.distributed as dist

    import paper_1601_07195_b200 as sv

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        p = world.bit_length() - 1
        d = dict(np.load(path + ".npz"))
        lay = sv.Layout(n, p, rank)
        m = lay.m
        shm = shared_memory.SharedMemory(create=True, size=16 << m, name=f"svp_{os.getpid()}_{rank}")
        amps = np.ndarray((1 << m,), dtype=np.complex128, buffer=shm.buf)
        amps[:] = d["init"][rank << m:(rank + 1) << m]
        state = ShmState(lay, amps, shm)
        ex = ShmOracleExecutor()
        fabric = sv.NvlinkFabric(fence="host", executor=ex)
        ops = [sv.GateOp(sv.GateMatrix.unchecked(q.reshape(2, 2)), int(t), None if c < 0 else int(c))
               for t, c, q in zip(d["t"], d["c"], d["q"])]
        plan = sv.plan_passes(ops, m, 0)
        for pz in plan:
            sv.execute_pass(state, pz, fabric)
        fabric.barrier()
        pids = fabric.exchange_objects(os.getpid())
        if rank == 0:
            parts = [amps.copy()]
            for r in range(1, world):
                other = shared_memory.SharedMemory(name=f"svp_{pids[r]}_{r}")
                parts.append(np.ndarray((1 << m,), dtype=np.complex128, buffer=other.buf).copy())
                other.close()
            np.savez(path + ".out.npz", full=np.concatenate(parts), nglobal=sum(not q.local for q in plan),
                     sent=fabric.sent_bytes)
        fabric.barrier()
        fabric.close()
        del amps
        shm.close()
        shm.unlink()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 9), (4, 10)])
def test_gloo_pass_fusion_matches_oracle(world, n):
    """QFT + random gates through plan_passes/execute_pass: global transform stages run as one
    exchange each (tags/fences/counters per stage) and the gathered state equals the oracle's."""
    import torch.multiprocessing as mp

    import paper_1601_07195_b200 as sv
    from conftest import random_state
    from oracle import oracle

    rng = np.random.default_rng(world * 100 + n)
    circ = sv.build_qft(n)
    circ.extend(sv.random_circuit(n, 40, rng, controlled_fraction=0.5).gates)
    init = random_state(rng, n)
    want = init.copy()
    oracle.run_circuit(want, circ.gates)
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "w")
        np.savez(path + ".npz", init=init, t=np.array([o.target for o in circ]),
                 c=np.array([-1 if o.control is None else o.control for o in circ]),
                 q=np.stack([o.gate.mat.reshape(4) for o in circ]))
        mp.spawn(_worker_passes, args=(world, _port(), path, n), nprocs=world, join=True)
        out = dict(np.load(path + ".out.npz"))
    assert np.array_equal(out["full"].view(np.uint64), want.view(np.uint64))
    m = n - (world.bit_length() - 1)
    stages = [p for p in sv.plan_passes(circ.gates, m) if p.kind == "global_stage"]
    assert len(stages) >= world.bit_length() - 1  # one exchange per global transform stage


def _worker_diag(rank, world, port, path, n):
    """NvlinkFabric(diagonal_local=True): diagonal global gates without an exchange."""
    import torch.distributed as dist

    import paper_1601_07195_b200 as sv

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        p = world.bit_length() - 1
        d = dict(np.load(path + ".npz"))
        lay = sv.Layout(n, p, rank)
        m = lay.m
        shm = shared_memory.SharedMemory(create=True, size=16 << m, name=f"svg_{os.getpid()}_{rank}")
        amps = np.ndarray((1 << m,), dtype=np.complex128, buffer=shm.buf)
        amps[:] = d["init"][rank << m:(rank + 1) << m]
        state = ShmState(lay, amps, shm)
        ex = ShmOracleExecutor()
        fabric = sv.NvlinkFabric(fence="host", executor=ex, diagonal_local=True)
        kinds = []
        for t, c, q in zip(d["t"], d["c"], d["q"]):
            t, c, gate = int(t), None if c < 0 else int(c), sv.GateMatrix.unchecked(q.reshape(2, 2))
            if max(t, -1 if c is None else c) < m:
                (ex.single(state, t, gate) if c is None else ex.controlled(state, c, t, gate))
            else:
                kinds.append(sv.plan_gate(lay, t, c, diag=sv.is_diagonal(gate)).kind)
                sv.apply_global(state, t, c, gate, fabric)
        fabric.barrier()
        pids = fabric.exchange_objects(os.getpid())
        if rank == 0:
            parts = [amps.copy()]
            for r in range(1, world):
                other = shared_memory.SharedMemory(name=f"svg_{pids[r]}_{r}")
                parts.append(np.ndarray((1 << m,), dtype=np.complex128, buffer=other.buf).copy())
                other.close()
            np.savez(path + ".out.npz", full=np.concatenate(parts), sent=fabric.sent_bytes,
                     ndiag=kinds.count("diag"), fences=fabric.fences)
        fabric.barrier()
        fabric.close()
        ex.cleanup()
        del amps
        shm.close()
        shm.unlink()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 8), (4, 9), (8, 10)])
def test_gloo_diagonal_local_protocol(world, n):
    """QFT + diagonal gates on global targets (cases 2, 5, 6) with diagonal_local=True: same state
    as the oracle; diagonal exchanges move no payload; every rank fences twice per global gate."""
    import torch.multiprocessing as mp

    import paper_1601_07195_b200 as sv
    from conftest import random_state
    from oracle import oracle

    p = world.bit_length() - 1
    m = n - p
    rng = np.random.default_rng(world * 7 + n)
    ops = list(sv.build_qft(n).gates)
    for k in range(6):
        q = sv.phase_r(k + 2) if k % 2 else sv.rotation_z(rng.uniform(0, 6))
        t = m + int(rng.integers(p))
        for c in [None, 0, m - 1] + [g for g in range(m, n) if g != t][:1]:
            ops.append(sv.GateOp(q, t, c))
    ops.append(sv.GateOp(sv.random_unitary(rng), n - 1))
    init = random_state(rng, n)
    want = init.copy()
    oracle.run_circuit(want, ops)
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "g")
        np.savez(path + ".npz", init=init, t=np.array([o.target for o in ops]),
                 c=np.array([-1 if o.control is None else o.control for o in ops]),
                 q=np.stack([o.gate.mat.reshape(4) for o in ops]))
        mp.spawn(_worker_diag, args=(world, _port(), path, n), nprocs=world, join=True)
        out = dict(np.load(path + ".out.npz"))
    assert np.array_equal(out["full"], want)
    glob = [o for o in ops if max(o.target, -1 if o.control is None else o.control) >= m]
    exch = [o for o in glob if o.target >= m and not sv.is_diagonal(o.gate)]
    assert int(out["ndiag"]) > 0
    # payload only for the non-diagonal exchanges (H stages of the QFT, the Haar gate): rank 0 takes part
    # in every uncontrolled one; none for the diagonal ones
    assert int(out["sent"]) <= sum(1 << (m + 4) for _ in exch)
    assert int(out["fences"]) == 2 * sum(1 for o in glob if o.target >= m) + 1


def _worker_remap(rank, world, port, path, n, plane="ipc"):
    """run_circuit_remapped: global<->local swaps instead of per-gate exchanges."""
    import torch.distributed as dist

    import paper_1601_07195_b200 as sv

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        p = world.bit_length() - 1
        d = dict(np.load(path + ".npz"))
        lay = sv.Layout(n, p, rank)
        m = lay.m
        shm = shared_memory.SharedMemory(create=True, size=16 << m, name=f"svr_{os.getpid()}_{rank}")
        amps = np.ndarray((1 << m,), dtype=np.complex128, buffer=shm.buf)
        amps[:] = d["init"][rank << m:(rank + 1) << m]
        state = ShmState(lay, amps, shm)
        ex = ShmOracleExecutor()
        fabric = sv.NvlinkFabric(fence="host", executor=ex, data_plane=plane, chunk_amps=1 << max(0, m - 4))
        circ = sv.Circuit(n, [sv.GateOp(sv.GateMatrix.unchecked(q.reshape(2, 2)), int(t), None if c < 0 else int(c))
                              for t, c, q in zip(d["t"], d["c"], d["q"])])
        qm = sv.run_circuit_remapped(state, circ, fabric, executor=ex)
        fabric.barrier()
        pids = fabric.exchange_objects(os.getpid())
        if rank == 0:
            parts = [amps.copy()]
            for r in range(1, world):
                other = shared_memory.SharedMemory(name=f"svr_{pids[r]}_{r}")
                parts.append(np.ndarray((1 << m,), dtype=np.complex128, buffer=other.buf).copy())
                other.close()
            np.savez(path + ".out.npz", full=np.concatenate(parts), sent=fabric.sent_bytes, ident=qm.identity)
        fabric.barrier()
        fabric.close()
        del amps
        shm.close()
        shm.unlink()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,plane", [(2, 8, "ipc"), (4, 9, "ipc"), (8, 10, "ipc"), (2, 8, "nccl"),
                                           (4, 9, "nccl")])
def test_gloo_remapped_execution(world, n, plane):
    """QFT + random gates with global<->local swaps over real ranks: the
    oracle's state, the identity map at the end, and fewer link bytes than the exchanges."""
    import torch.multiprocessing as mp

    import paper_1601_07195_b200 as sv
    from conftest import random_state
    from oracle import oracle

    p = world.bit_length() - 1
    m = n - p
    rng = np.random.default_rng(world * 11 + n)
    circ = sv.build_qft(n)
    circ.extend(sv.random_circuit(n, 60, rng, controlled_fraction=0.4).gates)
    init = random_state(rng, n)
    want = init.copy()
    oracle.run_circuit(want, circ.gates)
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "r")
        np.savez(path + ".npz", init=init, t=np.array([o.target for o in circ]),
                 c=np.array([-1 if o.control is None else o.control for o in circ]),
                 q=np.stack([o.gate.mat.reshape(4) for o in circ]))
        mp.spawn(_worker_remap, args=(world, _port(), path, n, plane), nprocs=world, join=True)
        out = dict(np.load(path + ".out.npz"))
    assert np.array_equal(out["full"], want) and bool(out["ident"])
    items, _ = sv.plan_remapped(circ.gates, n, m)
    assert int(out["sent"]) == sum(isinstance(i, sv.Swap) for i in items) << (m + 3)
    assert int(out["sent"]) < sum(1 for o in circ if o.target >= m) << (m + 4)
