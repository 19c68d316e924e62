"""Experiment: QFT top stages as one gathered-high-bit tile (k_tile with 4 register targets
above the tile) vs one same-target stage pass each.  Run under gpurun.

    python tools/exp_multistage.py [n]
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1601_07195_b200 as sv  # noqa: E402
from paper_1601_07195_b200 import _lib  # noqa: E402
from paper_1601_07195_b200.kernels import device_view, gate_array, stream_handle  # noqa: E402


def timed(fn, reps=3):
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


def group(a, ops, kind, tile=12):
    ptr, m = device_view(a)
    _lib.check(_lib.load().sv_apply_group(ptr, m, kind, gate_array(ops), len(ops), tile, stream_handle()))


n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
torch.cuda.set_device(0)
st = sv.init_random_state(sv.Layout(n), seed=1)
qft = sv.build_qft(n).gates
# split into same-target runs in order
runs = []
for op in qft:
    if runs and runs[-1][0].target == op.target:
        runs[-1].append(op)
    else:
        runs.append([op])
res = {"n": n, "first_targets": [r[0].target for r in runs[:6]]}
for k in (1, 2, 3, 4):
    ops = [op for r in runs[:k] for op in r]
    res[f"stages{k}_ms"] = timed(lambda: [group(st.amps, r, 2) for r in runs[:k]])
    res[f"tile{k}_ms"] = timed(lambda: group(st.amps, ops, 1))
print(json.dumps(res))
