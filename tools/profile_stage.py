"""ncu driver for the stage kernel (k_mstage): the QFT(n) pass plan, twice (second round profiled).

    ncu --set full --clock-control none --import-source on -k regex:k_mstage -s 10 -c 1 \
        -o gpurun_out/prof_mstage python tools/profile_stage.py 30
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1601_07195_b200 as sv  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
torch.cuda.set_device(0)
st = sv.init_random_state(sv.Layout(n), seed=1)
qft = sv.build_qft(n)
for _ in range(2):
    sv.run_circuit(st, qft, fusion=sv.FusionConfig(l_c=12, passes=True))
torch.cuda.synchronize()
print("ok")
