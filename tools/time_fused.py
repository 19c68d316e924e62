"""A/B timing of the fused kernels (run under gpurun): one same-target stage, one
random tile run, one diagonal-heavy tile run, and the QFT pass plan, at n qubits.

    python tools/time_fused.py [n] [reps]

Prints one JSON line of median milliseconds (CUDA events on the launch stream).
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1601_07195_b200 as sv  # noqa: E402


def timed(fn, reps):
    fn()
    out = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        out.append(s.elapsed_time(e))
    return float(np.median(out))


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    torch.cuda.set_device(0)
    st = sv.init_random_state(sv.Layout(n), seed=1)
    rng = np.random.default_rng(0)
    k = n - 2
    ctl = [c for c in range(n) if c != k][:29]
    stage = [sv.GateOp(sv.hadamard(), k)] + [sv.GateOp(sv.phase_r(j + 2), k, c) for j, c in enumerate(ctl)]
    tile = [sv.GateOp(sv.random_unitary(rng), int(rng.integers(12))) for _ in range(64)]
    tile_ctl = []
    for _ in range(64):
        t = int(rng.integers(12))
        c = None if rng.random() < 0.5 else int((t + 1 + rng.integers(n - 1)) % n)
        tile_ctl.append(sv.GateOp(sv.random_unitary(rng), t, c))
    diag = []
    for t in range(12):
        diag.append(sv.GateOp(sv.hadamard(), t))
        diag += [sv.GateOp(sv.phase_r(j + 2), t, c) for j, c in enumerate(range(t))]
    qft = sv.build_qft(n)
    fc = sv.FusionConfig(l_c=12, passes=True)
    res = {
        "n": n,
        "stage30_ms": timed(lambda: sv.kernels.apply_gates(st.amps, stage), reps),
        "tile64_random_ms": timed(lambda: sv.kernels.apply_gates(st.amps, tile, tile=12), reps),
        "tile64_ctl_ms": timed(lambda: sv.kernels.apply_gates(st.amps, tile_ctl, tile=12), reps),
        "tile_qft12_ms": timed(lambda: sv.kernels.apply_gates(st.amps, diag, tile=12), reps),
        "qft_ms": timed(lambda: sv.run_circuit(st, qft, fusion=fc), reps),
    }
    for lc in (12, 11, 10):
        steps = [[sv.GateOp(sv.random_unitary(rng), int(rng.integers(n))) for _ in range(25)] for _ in range(4)]
        fl = sv.FusionConfig(l_c=lc, passes=True)
        res[f"random25_lc{lc}_ms"] = timed(lambda: [sv.run_circuit(st, sv.Circuit(n, g), fusion=fl) for g in steps], reps) / 4
    csteps = []
    for _ in range(4):
        ops = []
        for _ in range(25):
            c, t = (int(x) for x in rng.choice(n, 2, replace=False))
            ops.append(sv.GateOp(sv.random_unitary(rng), t, c))
        csteps.append(ops)
    for lc in (12, 11):
        fl = sv.FusionConfig(l_c=lc, passes=True)
        res[f"controlled25_lc{lc}_ms"] = timed(
            lambda: [sv.run_circuit(st, sv.Circuit(n, g), fusion=fl) for g in csteps], reps) / 4
    f11 = sv.FusionConfig(l_c=11, passes=True)
    res["qft_lc11_ms"] = timed(lambda: sv.run_circuit(st, qft, fusion=f11), reps)
    b = sv.init_basis_state(sv.Layout(n), 5)
    res["qft_basis_ms"] = timed(lambda: sv.run_circuit(b, qft, fusion=fc), 1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
