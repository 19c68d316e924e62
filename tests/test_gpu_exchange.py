"""Global-qubit gates on the GPU: the fused NVLink exchange kernel and its host protocol.

The round's GPU box has ONE B200, so multi-rank runs are emulated two ways:

* loopback: all ranks' slices live on cuda:0 in one process and every rank's
  share of a gate runs in rank order on one stream.  The exchange kernel then
  reads/writes the partner slice through a plain device pointer instead of an
  IPC mapping -- same kernel, same indices, so it checks sv_exchange's
  arithmetic and pairing against the reference's distributed outputs;
* two processes on cuda:0 over gloo with real CUDA IPC mappings and host
  fences (no kernel ever waits on another), the product NvlinkFabric path
  end to end.
"""

from __future__ import annotations

import os
import socket
import tempfile

import numpy as np
import pytest
import torch

from conftest import golden_circuit, random_state

pytestmark = pytest.mark.gpu

sv = pytest.importorskip("paper_1601_07195_b200")
from oracle import oracle  # noqa: E402

DEV = "cuda:0"


class LoopbackFabric:
    """Fabric stand-in for ranks that share one process and one stream."""

    def __init__(self, states, rank):
        self.states, self.rank, self.num_ranks = states, rank, len(states)
        self.executor = sv.CudaExecutor()
        self.data_plane = "ipc"
        self.sent_bytes = self.received_bytes = 0
        self._tag = 0

    def fresh_tag(self):
        self._tag += 1
        return self._tag

    def barrier(self, state=None):
        pass

    def count(self, s, r):
        self.sent_bytes += s
        self.received_bytes += r

    def snapshot(self):
        return self.sent_bytes, self.received_bytes

    def ensure_registered(self, state):
        pass

    def peer_pointer(self, state, r):
        return self.states[r].amps.data_ptr()

    def reduce_sum(self, partial):
        raise NotImplementedError


def run_loopback(n, p, circ, full, fusion=None):
    states = [sv.state_from_global(sv.Layout(n, p, r), full, device=DEV) for r in range(1 << p)]
    fabrics = [LoopbackFabric(states, r) for r in range(1 << p)]
    deltas = np.zeros((1 << p, len(circ), 2), dtype=np.int64)
    if fusion is not None:
        plan = sv.plan_fusion(circ, fusion)
        for seg in plan.segments:
            for r in range(1 << p):
                sv.execute_plan(states[r], sv.FusionPlan(plan.l_c, [seg]), transport=fabrics[r])
    else:
        for gi, op in enumerate(circ):
            for r in range(1 << p):
                before = fabrics[r].snapshot()
                sv.apply_op(states[r], op, fabrics[r])
                after = fabrics[r].snapshot()
                deltas[r, gi] = (after[0] - before[0], after[1] - before[1])
    torch.cuda.synchronize()
    return np.concatenate([s.to_numpy() for s in states]), deltas


@pytest.mark.parametrize("name,n", [("mix8", 8), ("mix10", 10), ("ctl12", 12), ("single12", 12)])
@pytest.mark.parametrize("p", [1, 2, 3])
def test_loopback_matches_reference_distributed(golden, name, n, p):
    d = golden("circuits_small")
    circ = golden_circuit(d, name, n)
    full, deltas = run_loopback(n, p, circ, d[f"{name}_in"])
    assert np.array_equal(full, d[f"{name}_p{p}"])
    # per-gate, per-rank NVLink payload == the reference's CountingTransport deltas
    assert np.array_equal(deltas, d[f"{name}_p{p}_bytes"])


def test_loopback_fused_with_global_gates(golden):
    d = golden("circuits_small")
    circ = golden_circuit(d, "mix10", 10)
    full, _ = run_loopback(10, 2, circ, d["mix10_in"], fusion=sv.FusionConfig(l_c=5))
    assert np.array_equal(full, d["mix10_out"])


def test_loopback_every_exchange_case_n18():
    n, p = 18, 3
    m = n - p
    rng = np.random.default_rng(18)
    v = random_state(rng, n)
    ops = []
    for k in range(m, n):
        ops.append(sv.GateOp(sv.random_unitary(rng), k))
    for c, t in ((0, m), (1, m + 1), (m - 1, n - 1), (7, m + 2), (m, m + 1), (n - 1, m), (m + 1, 3), (n - 1, 0),
                 (0, n - 1), (m - 1, m)):
        ops.append(sv.GateOp(sv.random_unitary(rng), t, control=c))
    circ = sv.Circuit(n, ops)
    want = v.copy()
    oracle.run_circuit(want, ops, threads=8)
    got, _ = run_loopback(n, p, circ, v)
    assert np.array_equal(got, want)


def test_exchange_abi_rejects_bad_arguments():
    a = torch.zeros(16, dtype=torch.complex128, device=DEV)
    from paper_1601_07195_b200 import _lib

    q = sv.hadamard().qbuf()
    st = torch.cuda.current_stream().cuda_stream
    L = _lib.load()
    assert L.sv_exchange(a.data_ptr(), a.data_ptr(), 4, 1, -1, q, st) == _lib.SV_EINVAL
    assert L.sv_exchange(a.data_ptr(), a.data_ptr() + 8, 4, 1, -1, q, st) == _lib.SV_EINVAL
    assert L.sv_exchange(a.data_ptr(), 0, 4, 1, -1, q, st) == _lib.SV_EINVAL


@pytest.mark.parametrize("c_local", [-1, 0, 2, 5])
def test_exchange_chunk_staged_protocol(c_local):
    """The NCCL data plane's chunk step, with the send/recv replaced by device copies."""
    from paper_1601_07195_b200 import _lib

    n, m = 12, 11
    rng = np.random.default_rng(40 + c_local)
    v = random_state(rng, n)
    q = sv.random_unitary(rng)
    want = v.copy()
    if c_local < 0:
        oracle.apply_single(want, n - 1, q)
    else:
        oracle.apply_controlled(want, c_local, n - 1, q)
    ranks = [torch.from_numpy(v[: 1 << m].copy()).to(DEV), torch.from_numpy(v[1 << m:].copy()).to(DEV)]
    half, chunk = 1 << (m - 1), 1 << (m - 3)
    L = _lib.load()
    st = torch.cuda.current_stream().cuda_stream
    for stage in (0, 1):
        comp, pas = ranks[stage], ranks[1 - stage]  # zero side computes the first half
        for j0 in range(stage * half, (stage + 1) * half, chunk):
            buf = pas[j0:j0 + chunk].clone()          # "recv" the partner's chunk
            _lib.check(L.sv_exchange_chunk(comp.data_ptr(), buf.data_ptr(), m, int(stage == 0), c_local, q.qbuf(),
                                           j0, chunk, st))
            pas[j0:j0 + chunk].copy_(buf)             # "send" it back
    torch.cuda.synchronize()
    assert np.array_equal(np.concatenate([r.cpu().numpy() for r in ranks]), want)
    with pytest.raises(ValueError):
        _lib.check(L.sv_exchange_chunk(ranks[0].data_ptr(), buf.data_ptr(), m, 1, c_local if c_local > 0 else 1,
                                       q.qbuf(), 1, chunk, st))  # misaligned start


# --------------------------------------------------- two processes, real IPC


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ipc_worker(rank, world, port, path, n, plane):
    import torch.distributed as dist

    import paper_1601_07195_b200 as svm

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        p = world.bit_length() - 1
        d = dict(np.load(path + ".in.npz"))
        fabric = svm.NvlinkFabric(fence="host", data_plane=plane, chunk_amps=1 << 7)
        circ = svm.Circuit(n, [svm.GateOp(svm.GateMatrix.unchecked(q.reshape(2, 2)), int(t),
                                          None if c < 0 else int(c)) for t, c, q in zip(d["t"], d["c"], d["q"])])
        st = svm.state_from_global(svm.Layout(n, p, rank), d["init"], device="cuda:0")
        recs = svm.run_circuit(st, circ, fabric, record=True)
        full = svm.gather_full_state(st, fabric)
        norm = svm.global_norm_sq(st, fabric)
        if rank == 0:
            np.savez(path + ".out.npz", full=full, norm=norm, sent=fabric.sent_bytes, recv=fabric.received_bytes,
                     nrec=len(recs))
        fabric.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("plane", ["ipc", "nccl", "ce"])
def test_two_process_ipc_fabric_matches_oracle(plane):
    import torch.multiprocessing as mp

    n, world = 12, 2
    rng = np.random.default_rng(31)
    init = random_state(rng, n)
    circ = sv.random_circuit(n, 80, np.random.default_rng(32), controlled_fraction=0.4)
    circ.extend([sv.GateOp(sv.random_unitary(rng), n - 1), sv.GateOp(sv.random_unitary(rng), n - 1, control=0),
                 sv.GateOp(sv.random_unitary(rng), 2, control=n - 1)])
    want = init.copy()
    oracle.run_circuit(want, circ.gates)
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "ipc")
        np.savez(path + ".in.npz", init=init, t=np.array([o.target for o in circ]),
                 c=np.array([-1 if o.control is None else o.control for o in circ]),
                 q=np.stack([o.gate.mat.reshape(4) for o in circ]))
        mp.spawn(_ipc_worker, args=(world, _free_port(), path, n, plane), nprocs=world, join=True)
        out = dict(np.load(path + ".out.npz"))
    assert np.array_equal(out["full"], want)
    assert abs(float(out["norm"]) - 1.0) < 1e-12
    m = n - 1
    n_exch = sum(1 for o in circ if o.max_qubit() >= m and not (o.control is not None and o.target < m))
    assert int(out["nrec"]) == len(circ)
    assert int(out["sent"]) == int(out["recv"]) > 0
    assert n_exch >= 3


@pytest.mark.parametrize("p", [1, 2, 3])
@pytest.mark.parametrize("fused", [False, True])
def test_inproc_copy_engine_plane_matches_oracle(p, fused):
    """data_plane="ce": peer chunks copied in (cudaMemcpyAsync, copy-in stream), updated by the
    exchange kernel, pushed back (copy-out stream), double-buffered; chunks smaller than
    2^(c+1) for high local controls; stage exchanges run per gate on this plane."""
    n = 14
    m = n - p
    rng = np.random.default_rng(50 + p)
    v = random_state(rng, n)
    circ = sv.build_qft(n)
    circ.extend(sv.random_circuit(n, 60, np.random.default_rng(p), controlled_fraction=0.5).gates)
    circ.extend([sv.GateOp(sv.random_unitary(rng), n - 1, control=c) for c in (0, 3, m - 2, m - 1)])
    want = v.copy()
    oracle.run_circuit(want, circ.gates, threads=8)
    sts = [sv.LocalState(sv.Layout(n, p, r), torch.from_numpy(v[r << m:(r + 1) << m].copy()).to(DEV))
           for r in range(1 << p)]
    fabs = sv.InprocFabric.group(sts, data_plane="ce", chunk_amps=1 << 6)
    sv.run_circuit_inproc(sts, circ, fabs, fusion=sv.FusionConfig(l_c=10, passes=True) if fused else None)
    torch.cuda.synchronize()
    got = np.concatenate([s.to_numpy() for s in sts])
    assert np.array_equal(got, want)


def test_copy_engine_plane_scratch_accounting():
    """The staged planes draw their two chunk buffers from the caller's ScratchPool: the
    reference's high-water bound 2 * chunk * 16 B (distributed.py:161-181)."""
    n, p = 12, 1
    m = n - p
    v = random_state(np.random.default_rng(5), n)
    sts = [sv.LocalState(sv.Layout(n, p, r), torch.from_numpy(v[r << m:(r + 1) << m].copy()).to(DEV))
           for r in range(2)]
    fabs = sv.InprocFabric.group(sts, data_plane="ce", chunk_amps=1 << 20)
    pool = sv.ScratchPool()
    q = sv.random_unitary(np.random.default_rng(6))
    for r in range(2):
        sv.apply_single_distributed(sts[r], n - 1, q, fabs[r], chunk_amps=1 << 7, scratch=pool)
    torch.cuda.synchronize()
    want = v.copy()
    oracle.apply_single(want, n - 1, q.mat)
    assert np.array_equal(np.concatenate([s.to_numpy() for s in sts]), want)
    assert pool.high_water_bytes == 2 * (1 << 7) * 16 and pool.outstanding_bytes == 0
