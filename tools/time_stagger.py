"""Times the exact pass-fused workloads (config-4-shape random steps, a 16-gate tile, QFT): the
A/B timing behind tools/ab_qft.sh.  (Written for the first-wave stagger experiment of round 2 --
profiles/r02_probes.md section 3; the SVB_TILE_STAGGER / SVB_MS_STAGGER switches it echoed no
longer exist in the library.)

    python tools/time_stagger.py [n] [reps]
"""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1601_07195_b200 as sv  # noqa: E402
from tools.time_fused import timed  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    torch.cuda.set_device(0)
    st = sv.init_random_state(sv.Layout(n), seed=1)
    rng = np.random.default_rng(0)
    res = {"tile": os.environ.get("SVB_TILE_STAGGER", "0"), "ms": os.environ.get("SVB_MS_STAGGER", "0")}
    steps = [[sv.GateOp(sv.random_unitary(rng), int(rng.integers(n))) for _ in range(25)] for _ in range(4)]
    fl = sv.FusionConfig(l_c=12, passes=True)
    res["random25_ms"] = round(timed(lambda: [sv.run_circuit(st, sv.Circuit(n, g), fusion=fl) for g in steps], reps) / 4, 3)
    tile = [sv.GateOp(sv.random_unitary(rng), int(rng.integers(12))) for _ in range(16)]
    res["tile16_ms"] = round(timed(lambda: sv.kernels.apply_gates(st.amps, tile, tile=12), reps), 3)
    qft = sv.build_qft(n)
    res["qft_ms"] = round(timed(lambda: sv.run_circuit(st, qft, fusion=fl), reps), 3)
    print(json.dumps(res))


main()
