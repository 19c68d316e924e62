"""k_tile phase probe: G general gates per pass with (a) targets on the natural register bits
(no transposes), (b) targets on the low four bits (one transpose in, one out), (c) alternating
register sets (a transpose per gate), at n qubits.  Prints ms per pass next to the HBM pass time
and the FP64 floor so the overlap (or its absence) is visible.

    python tools/tile_probe2.py [n] [reps]
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1601_07195_b200 as sv  # noqa: E402
from tools.time_fused import timed  # noqa: E402
from paper_1601_07195_b200 import _lib  # noqa: E402
from paper_1601_07195_b200.kernels import device_view, gate_array, stream_handle  # noqa: E402


def tile_group(amps, ops, T):
    ptr, m = device_view(amps)
    _lib.check(_lib.load().sv_apply_group(ptr, m, 1, gate_array(ops), len(ops), T, stream_handle()))


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    T = int(sys.argv[3]) if len(sys.argv) > 3 else 12
    torch.cuda.set_device(0)
    st = sv.init_random_state(sv.Layout(n), seed=1)
    rng = np.random.default_rng(0)
    out = {"n": n, "T": T}
    out["single_ms"] = round(timed(lambda: sv.kernels.apply_gates(st.amps, [sv.GateOp(sv.random_unitary(rng), n - 1)]), reps), 3)
    for G in (1, 2, 4, 8, 12, 16, 32):
        nat = [sv.GateOp(sv.random_unitary(rng), T - 4 + (i % 4)) for i in range(G)]
        low = [sv.GateOp(sv.random_unitary(rng), i % 4) for i in range(G)]
        alt = [sv.GateOp(sv.random_unitary(rng), (i * 4 + (i // 3)) % T) for i in range(G)]
        out[f"nat{G}"] = round(timed(lambda: tile_group(st.amps, nat, T), reps), 3)
        out[f"low{G}"] = round(timed(lambda: tile_group(st.amps, low, T), reps), 3)
        out[f"alt{G}"] = round(timed(lambda: tile_group(st.amps, alt, T), reps), 3)
    print(json.dumps(out))


main()
