"""Controlled-gate launches for an ncu capture (run under gpurun, one GPU): at n qubits, after the
state init, the controlled gates (c, t) = (5, 17), (1, 17), (0, 17), (2, 17), (3, 17) -- the DRAM
regimes of sv_apply_controlled (control runs >= 128 B; 32/64-B runs inside 128-B lines; 16-B
interleave, MODE_PRED; 64-B and 128-B runs).  profiles/run_ncu_controlled.sh captures them.

    python tools/profile_controlled.py [n]
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1601_07195_b200 as sv  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
    torch.cuda.set_device(0)
    st = sv.init_random_state(sv.Layout(n), seed=0)
    q = sv.random_unitary(np.random.default_rng(1))
    torch.cuda.synchronize()
    for c, t in ((5, 17), (1, 17), (0, 17), (2, 17), (3, 17)):
        sv.apply_controlled_local(st, c, t, q)
    torch.cuda.synchronize()
    print("ok", n)


if __name__ == "__main__":
    main()
