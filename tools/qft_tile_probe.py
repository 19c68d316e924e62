"""Transform stages as register tiles vs stage passes (run under gpurun): the first k
stages of build_qft(n) (targets n-1 .. n-k) through one k_tile pass that gathers the k
targets (sv_apply_group SV_GROUP_TILE), against the same gates as four-target k_mstage
passes.  Prints one JSON line of median milliseconds (CUDA events) and the max |diff|
between the two results (bitwise expected).

    python tools/qft_tile_probe.py [n] [reps]
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1601_07195_b200 as sv  # noqa: E402
from paper_1601_07195_b200 import _lib  # noqa: E402
from paper_1601_07195_b200.core import device_view  # noqa: E402
from paper_1601_07195_b200.kernels import gate_array, stream_handle  # noqa: E402


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


def group(st, kind, ops, tile=12):
    ptr, m = device_view(st.amps)
    _lib.check(_lib.load().sv_apply_group(ptr, m, kind, gate_array(ops), len(ops), tile, stream_handle()))


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    torch.cuda.set_device(0)
    qft = sv.build_qft(n).gates
    res = {"n": n}
    a = sv.init_random_state(sv.Layout(n), seed=1)
    b = sv.init_random_state(sv.Layout(n), seed=1)
    for k in (4, 8):
        ops = [op for op in qft if op.target >= n - k]
        stages = [[op for op in ops if n - 4 * (i + 1) <= op.target < n - 4 * i] for i in range(k // 4)]
        res[f"stages{k}_gates"] = len(ops)
        res[f"stages{k}_tile_ms"] = timed(lambda: group(a, _lib.SV_GROUP_TILE, ops), reps)
        res[f"stages{k}_mstage_ms"] = timed(lambda: [group(b, _lib.SV_GROUP_STAGE, s, 0) for s in stages], reps)
    res["max_abs_diff"] = float((a.amps - b.amps).abs().max())
    print(json.dumps(res))


if __name__ == "__main__":
    main()
