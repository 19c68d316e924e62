"""Generate the golden fixtures from the reference implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package from /root/reference/pkg/src (read-only,
never copied) and records its inputs and outputs as small .npz fixtures.  The
GPU box has no /root/reference; the tests there read only these files.

Every fixture stores the gate matrices explicitly (np.linalg.qr may round
differently on another CPU) and every input state explicitly or, for the n=20
parity config, as (rng seed, stored L2 norm, sha256 of the normalised input)
so the box can rebuild the identical input with numpy's platform-independent
PCG64 stream and a plain elementwise division.
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

import svsim  # noqa: E402  (reference, imported read-only)
from svsim import (  # noqa: E402
    CountingTransport,
    FusionConfig,
    GateOp,
    Layout,
    apply_op,
    build_iqft,
    build_qft,
    gather_full_state,
    init_basis_state,
    random_circuit,
    random_unitary,
    run_circuit,
    run_spmd,
    state_from_global,
)
from svsim.kernels import apply_controlled_raw, apply_single_raw  # noqa: E402

OUT = Path(__file__).resolve().parent


def random_state(rng, n):
    # recipe of pkg/tests/test_kernels.py:32-34
    v = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    return (v / np.linalg.norm(v)).astype(np.complex128)


def pack_circuit(circ):
    t = np.array([op.target for op in circ.gates], dtype=np.int32)
    c = np.array([-1 if op.control is None else op.control for op in circ.gates], dtype=np.int32)
    q = np.stack([op.gate.mat.reshape(4) for op in circ.gates]).astype(np.complex128)
    return t, c, q


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def serial(circ, init, **kw):
    st = state_from_global(Layout(circ.n, 0, 0), init)
    run_circuit(st, circ, **kw)
    return st.amps.copy()


def spmd(circ, p, init, chunk_amps=None):
    def worker(rank, transport):
        counting = CountingTransport(transport)
        st = state_from_global(Layout(circ.n, p, rank), init)
        deltas = []
        before = counting.snapshot()
        for op in circ.gates:
            apply_op(st, op, counting, chunk_amps=chunk_amps)
            after = counting.snapshot()
            deltas.append((after[0] - before[0], after[1] - before[1]))
            before = after
        return gather_full_state(st, counting), np.array(deltas, dtype=np.int64)

    res = run_spmd(1 << p, worker)
    return res[0][0], np.stack([r[1] for r in res])


def kernels_n5():
    rng = np.random.default_rng(1234)
    n = 5
    ins, qs, outs, kinds = [], [], [], []
    for k in range(n):
        v = random_state(rng, n)
        q = random_unitary(rng)
        w = v.copy()
        apply_single_raw(w, k, q)
        ins.append(v), qs.append(q.mat.reshape(4)), outs.append(w), kinds.append((-1, k))
    for c in range(n):
        for t in range(n):
            if c == t:
                continue
            v = random_state(rng, n)
            q = random_unitary(rng)
            w = v.copy()
            apply_controlled_raw(w, c, t, q)
            ins.append(v), qs.append(q.mat.reshape(4)), outs.append(w), kinds.append((c, t))
    np.savez_compressed(OUT / "kernels_n5.npz", inp=np.stack(ins), q=np.stack(qs), out=np.stack(outs),
                        ct=np.array(kinds, dtype=np.int32))


def circuits_small():
    """Random mixed circuits: unfused, fused, and distributed (p=1,2,3) outputs."""
    data = {}
    for name, n, g, frac, seed in (("mix10", 10, 120, 0.3, 7), ("ctl12", 12, 100, 1.0, 11),
                                   ("single12", 12, 100, 0.0, 13), ("mix8", 8, 100, 0.3, 8)):
        rng = np.random.default_rng(seed)
        circ = random_circuit(n, g, rng, controlled_fraction=frac)
        init = random_state(np.random.default_rng(seed + 100), n)
        t, c, q = pack_circuit(circ)
        data[f"{name}_t"], data[f"{name}_c"], data[f"{name}_q"] = t, c, q
        data[f"{name}_in"] = init
        data[f"{name}_out"] = serial(circ, init)
        for l_c in (3, 6):
            data[f"{name}_fused{l_c}"] = serial(circ, init, fusion=FusionConfig(l_c=l_c))
        for p in (1, 2, 3):
            full, deltas = spmd(circ, p, init)
            data[f"{name}_p{p}"] = full
            data[f"{name}_p{p}_bytes"] = deltas
    np.savez_compressed(OUT / "circuits_small.npz", **data)


def transforms():
    data = {}
    for n in (10, 12):
        init = random_state(np.random.default_rng(500 + n), n)
        for name, circ in (("qft", build_qft(n)), ("iqft", build_iqft(n))):
            t, c, q = pack_circuit(circ)
            data[f"{name}{n}_t"], data[f"{name}{n}_c"], data[f"{name}{n}_q"] = t, c, q
            data[f"{name}{n}_in"] = init
            data[f"{name}{n}_out"] = serial(circ, init)
            data[f"{name}{n}_fused5"] = serial(circ, init, fusion=FusionConfig(l_c=5))
    # basis input 5 through QFT(8): closed form available too
    data["qft8_basis5"] = serial(build_qft(8), np.eye(1, 256, 5, dtype=np.complex128)[0])
    np.savez_compressed(OUT / "transforms.npz", **data)


def config1():
    """BASELINE config 1: n=20, 200 Haar single-qubit gates, seeds (state 0, circuit 1)."""
    n = 20
    rng0 = np.random.default_rng(0)
    raw = rng0.standard_normal(1 << n) + 1j * rng0.standard_normal(1 << n)
    norm = float(np.linalg.norm(raw))
    init = (raw / norm).astype(np.complex128)
    circ = random_circuit(n, 200, np.random.default_rng(1), controlled_fraction=0.0)
    t, c, q = pack_circuit(circ)
    out = serial(circ, init)
    fused = serial(circ, init, fusion=FusionConfig(l_c=12))
    idx = np.random.default_rng(99).choice(1 << n, size=4096, replace=False).astype(np.int64)
    np.savez_compressed(
        OUT / "config1_n20.npz", t=t, c=c, q=q, norm=np.float64(norm), in_sha=sha(init),
        out_sha=sha(out), fused_sha=sha(fused), idx=idx, out_sample=out[idx], n=np.int32(n),
    )


def known_answers():
    data = {}
    # CNOT truth table (pkg/tests/test_kernels.py:78-85)
    for g in range(4):
        v = np.zeros(4, complex)
        v[g] = 1.0
        apply_controlled_raw(v, 0, 1, svsim.pauli_x())
        data[f"cnot_{g}"] = v
    # X across the rank boundary (pkg/tests/test_distributed.py:95-100)
    full = random_state(np.random.default_rng(3), 2)
    out, _ = spmd(svsim.Circuit(2, [GateOp(svsim.pauli_x(), 1)]), 1, full)
    data["xswap_in"], data["xswap_out"] = full, out
    # basis-state norms / probabilities (core.py:147-167)
    st = init_basis_state(Layout(6, 0, 0), 37)
    run_circuit(st, random_circuit(6, 30, np.random.default_rng(4)))
    data["prob_state"] = st.amps.copy()
    data["prob_bits"] = np.array([svsim.probability_of_bit(st, b) for b in range(6)])
    data["prob_norm"] = np.float64(svsim.global_norm_sq(st))
    np.savez_compressed(OUT / "known_answers.npz", **data)


if __name__ == "__main__":
    kernels_n5()
    circuits_small()
    transforms()
    config1()
    known_answers()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)
