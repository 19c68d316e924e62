"""Small driver for ncu captures of the fused kernels (run under gpurun; see profiles/run_ncu_fused.sh).

    python tools/profile_kernels.py [n] [what]

what = tile64: one 64-gate random run on targets < 12 (k_tile<12, false>);
       qft:    the QFT(n) pass plan (at n = 28: six k_mstage passes of four transform
               stages each, then the k_tile<12, true> tail);
       random: the bench's config-4-shape step, 25 Haar gates on uniform targets, pass plan
               (k_tile runs that gather up to four high qubits, ~6.5 gates per pass);
       all (default): the three in that order.
Two rounds; profile the second (ncu -s skips the first round's launches).
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1601_07195_b200 as sv  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
what = sys.argv[2] if len(sys.argv) > 2 else "all"
torch.cuda.set_device(0)
st = sv.init_random_state(sv.Layout(n), seed=1)
rng = np.random.default_rng(0)
tile = [sv.GateOp(sv.random_unitary(rng), int(rng.integers(12))) for _ in range(64)]
qft = sv.build_qft(n)
rand = sv.random_circuit(n, 25, np.random.default_rng(1), controlled_fraction=0.0)
fc = sv.FusionConfig(l_c=12, passes=True)
for _ in range(2):
    if what in ("all", "tile64"):
        sv.kernels.apply_gates(st.amps, tile, tile=12)
    if what in ("all", "qft"):
        sv.run_circuit(st, qft, fusion=fc)
    if what in ("all", "random"):
        sv.run_circuit(st, rand, fusion=fc)
    if what == "qft_tol":  # tolerance planner: k_dstage2 passes, then k_dlow
        sv.run_circuit(st, qft, fusion=sv.FusionConfig(l_c=12, passes=True, exact=False))
torch.cuda.synchronize()
plan = sv.plan_passes(rand.gates, n, 12)
print("ok; random plan:", [(p.kind, len(p.gates)) for p in plan])
