"""Small driver for ncu captures of the fused kernels (run under gpurun; see profiles/run_ncu_fused.sh)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1601_07195_b200 as sv  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
torch.cuda.set_device(0)
st = sv.init_random_state(sv.Layout(n), seed=1)
rng = np.random.default_rng(0)
k = n - 2
ctl = [c for c in range(n) if c != k][:29]
stage = [sv.GateOp(sv.hadamard(), k)] + [sv.GateOp(sv.phase_r(j + 2), k, c) for j, c in enumerate(ctl)]
tile = [sv.GateOp(sv.random_unitary(rng), int(rng.integers(12))) for _ in range(64)]
qft_tail = [op for op in sv.build_qft(n).gates if op.target < 12]
for _ in range(2):
    sv.kernels.apply_gates(st.amps, stage)
    sv.kernels.apply_gates(st.amps, tile, tile=12)
    sv.kernels.apply_gates(st.amps, qft_tail, tile=12)
torch.cuda.synchronize()
print("ok")
