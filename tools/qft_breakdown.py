"""Per-pass device time of the QFT(n) pass plan (run under gpurun).

    python tools/qft_breakdown.py [n] [l_c]

One line per pass: kind, gate count, target, ms (CUDA events), then the total.
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1601_07195_b200 as sv  # noqa: E402
from paper_1601_07195_b200.passes import plan_passes, tile_for  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
l_c = int(sys.argv[2]) if len(sys.argv) > 2 else 12
torch.cuda.set_device(0)
st = sv.init_random_state(sv.Layout(n), seed=1)
qft = sv.build_qft(n)
fc = sv.FusionConfig(l_c=l_c, passes=True)
sv.run_circuit(st, qft, fusion=fc)
recs = sv.run_circuit(st, qft, fusion=fc, record=True)
plan = plan_passes(qft.gates, n, tile_for(l_c, n))
tot = 0.0
for p, r in zip(plan, recs):
    ms = r.seconds * 1e3
    tot += ms
    print(f"{p.kind:14s} gates={len(p.gates):3d} target={p.target!s:5s} {ms:8.3f} ms")
print(f"total {tot:.2f} ms over {len(recs)} passes")
