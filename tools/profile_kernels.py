"""Small driver for ncu captures of the fused kernels (run under gpurun; see profiles/run_ncu_fused.sh).

Launch order (for ncu -k/-s/-c), per round: one 64-gate random run on targets < 12
(k_tile<12, false>), then the QFT(n) pass plan (at n = 28: eight k_mstage passes of three
transform stages each, then one k_tile<12, true> tail).  Two rounds; profile the second.
"""
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
tile = [sv.GateOp(sv.random_unitary(rng), int(rng.integers(12))) for _ in range(64)]
qft = sv.build_qft(n)
for _ in range(2):
    sv.kernels.apply_gates(st.amps, tile, tile=12)
    sv.run_circuit(st, qft, fusion=sv.FusionConfig(l_c=12, passes=True))
torch.cuda.synchronize()
print("ok")
