"""Per-placement throughput sweep on one GPU (diagnostics; bench.py is the contract).

    python tools/gate_sweep.py [--n 30] [--reps 5] [--what single,controlled,fused,qft,config1]

Prints one JSON object per measurement: kernel class, placement, median ms, GB/s against the
reference's algorithmic accounting (32*2^m single, 16*2^m controlled, 32*2^m physical for a
fused run plus G*32*2^m effective).
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1601_07195_b200 as sv  # noqa: E402


def timeit(fn, reps):
    st = torch.cuda.current_stream()
    ts = []
    for _ in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts[1:]))


def emit(**kw):
    print(json.dumps(kw), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--what", default="single,controlled,fused,qft,config1")
    a = ap.parse_args()
    what = set(a.what.split(","))
    n = a.n
    torch.cuda.set_device(0)
    st = sv.init_random_state(sv.Layout(n), seed=1)
    rng = np.random.default_rng(0)
    q = sv.random_unitary(rng)
    if "single" in what:
        for k in range(n):
            ms = timeit(lambda: sv.apply_single_raw(st.amps, k, q), a.reps)
            emit(kind="single", k=k, ms=round(ms, 4), gbps=round((32 << n) / ms / 1e6, 1))
    if "controlled" in what:
        pairs = [(c, t) for c in (0, 1, 2, 3, 4, 5, 6, 10, 15, 20, n - 2, n - 1)
                 for t in (0, 1, 2, 4, 5, 8, 15, n - 1) if c != t and c < n and t < n]
        for c, t in pairs:
            ms = timeit(lambda: sv.apply_controlled_raw(st.amps, c, t, q), a.reps)
            emit(kind="controlled", c=c, t=t, ms=round(ms, 4), gbps=round((16 << n) / ms / 1e6, 1))
    if "fused" in what:
        for G in (1, 2, 4, 8, 16, 32, 64):
            for lmax in (5, 12, 13):
                gates = [sv.GateOp(sv.random_unitary(rng), int(rng.integers(lmax))) for _ in range(G)]
                ms = timeit(lambda: sv.run_fused(st, gates, lmax), a.reps)
                emit(kind="fused", gates=G, lmax=lmax, ms=round(ms, 4), phys_gbps=round((32 << n) / ms / 1e6, 1),
                     eff_gbps=round(G * (32 << n) / ms / 1e6, 1))
    if "tile" in what:
        for G in (1, 4, 16, 64):
            for T in (12, 13):
                gates = [sv.GateOp(sv.random_unitary(rng), int(rng.integers(T))) for _ in range(G)]
                ms = timeit(lambda: sv.kernels.apply_gates(st.amps, gates, tile=T), a.reps)
                emit(kind="tile", gates=G, T=T, ms=round(ms, 4), phys_gbps=round((32 << n) / ms / 1e6, 1),
                     eff_gbps=round(G * (32 << n) / ms / 1e6, 1))
        for k in (13, 20, n - 1):
            for G in (2, 8, 30):
                gates = [sv.GateOp(sv.hadamard(), k)] + [sv.GateOp(sv.phase_r(j + 2), k, (k + 1 + j) % n)
                                                          for j in range(G - 1)]
                ms = timeit(lambda: sv.kernels.apply_gates(st.amps, gates), a.reps)
                emit(kind="stage", k=k, gates=G, ms=round(ms, 4), phys_gbps=round((32 << n) / ms / 1e6, 1))
    if "exchange" in what:
        # loopback: both "ranks" on this GPU, so the partner slice is local HBM -- this checks
        # the exchange kernels' own efficiency (HBM-bound here; NVLink-bound across GPUs)
        from paper_1601_07195_b200 import _lib

        m = n - 1
        ta = torch.empty(1 << m, dtype=torch.complex128, device="cuda")
        tb = torch.empty(1 << m, dtype=torch.complex128, device="cuda")
        ta.copy_(st.amps[: 1 << m])
        tb.copy_(st.amps[1 << m:])
        L = _lib.load()
        s = torch.cuda.current_stream().cuda_stream
        for c_local in (-1, 0, 3, m - 1):
            ms = timeit(lambda: (_lib.check(L.sv_exchange(ta.data_ptr(), tb.data_ptr(), m, 1, c_local, q.qbuf(), s)),
                                 _lib.check(L.sv_exchange(tb.data_ptr(), ta.data_ptr(), m, 0, c_local, q.qbuf(), s))),
                        a.reps)
            touched = (32 << m) if c_local < 0 else (16 << m)
            emit(kind="exchange_loopback", c_local=c_local, ms=round(ms, 4),
                 hbm_gbps=round(2 * touched / ms / 1e6, 1))
        stage = [sv.GateOp(sv.hadamard(), n - 1)] + [sv.GateOp(sv.phase_r(j + 2), n - 1, j) for j in range(20)]
        ga = sv.kernels.gate_array(stage)
        ms = timeit(lambda: (_lib.check(L.sv_exchange_stage(ta.data_ptr(), tb.data_ptr(), m, 1, ga, len(stage), s)),
                             _lib.check(L.sv_exchange_stage(tb.data_ptr(), ta.data_ptr(), m, 0, ga, len(stage), s))),
                    a.reps)
        emit(kind="exchange_stage_loopback", gates=len(stage), ms=round(ms, 4),
             hbm_gbps=round(2 * (32 << m) / ms / 1e6, 1))
        del ta, tb
    if "qft" in what:
        circ = sv.build_qft(n)
        for l_c in (None, 12, 13, "p12", "p13"):
            if isinstance(l_c, str):
                fusion = sv.FusionConfig(l_c=int(l_c[1:]), passes=True)
            else:
                fusion = None if l_c is None else sv.FusionConfig(l_c=l_c)
            ms = timeit(lambda: sv.run_circuit(st, circ, fusion=fusion), max(1, a.reps // 2))
            eff = sum((32 if op.control is None else 16) << n for op in circ)
            emit(kind="qft", n=n, l_c=l_c, gates=len(circ), ms=round(ms, 3), eff_gbps=round(eff / ms / 1e6, 1),
                 ms_per_gate=round(ms / len(circ), 4))
    if "config1" in what:
        m = 20
        s20 = sv.init_random_state(sv.Layout(m), seed=2)
        circ = sv.random_circuit(m, 200, np.random.default_rng(1), controlled_fraction=0.0)
        for l_c in (None, 12, 13, "p13"):
            if isinstance(l_c, str):
                fusion = sv.FusionConfig(l_c=int(l_c[1:]), passes=True)
            else:
                fusion = None if l_c is None else sv.FusionConfig(l_c=l_c)
            ms = timeit(lambda: sv.run_circuit(s20, circ, fusion=fusion), a.reps)
            emit(kind="config1", n=m, l_c=l_c, gates=200, ms=round(ms, 3), us_per_gate=round(ms * 1e3 / 200, 2),
                 eff_gbps=round(200 * (32 << m) / ms / 1e6, 1))
        for l_c in (None, 13):
            fusion = None if l_c is None else sv.FusionConfig(l_c=l_c, passes=True)
            g = sv.CircuitGraph(s20, circ, fusion=fusion)
            ms = timeit(g.replay, a.reps)
            emit(kind="config1_graph", n=m, passes=l_c, gates=200, ms=round(ms, 3),
                 us_per_gate=round(ms * 1e3 / 200, 2), eff_gbps=round(200 * (32 << m) / ms / 1e6, 1))


if __name__ == "__main__":
    main()
