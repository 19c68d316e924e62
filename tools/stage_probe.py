"""Time single k_mstage launches of different compositions (run under gpurun).

    python tools/stage_probe.py [n] [reps]
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
    return round(float(np.median(out)), 3)


def qft_stages(n, targets):
    ops = []
    for i in targets:
        ops.append(sv.GateOp(sv.hadamard(), i))
        ops += [sv.GateOp(sv.phase_r(i - c + 1), i, c) for c in range(i - 1, -1, -1)]
    return ops


n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
torch.cuda.set_device(0)
st = sv.init_random_state(sv.Layout(n), seed=1)
ptr, m = device_view(st.amps)
L = _lib.load()


def stage(ops):
    arr = gate_array(ops)
    return lambda: _lib.check(L.sv_apply_group(ptr, m, _lib.SV_GROUP_STAGE, arr, len(ops), 0, stream_handle()))


cases = {
    "s1_hi_H+29CR": qft_stages(n, [n - 2])[:30],
    "s1_lo_H+29CR": [sv.GateOp(sv.hadamard(), 7)] + [sv.GateOp(sv.phase_r(2 + j), 7, c)
                                                     for j, c in enumerate([c for c in range(n) if c != 7][:29])],
    "q4_hi": qft_stages(n, range(n - 1, n - 5, -1)),
    "q4_hi_noH": [o for o in qft_stages(n, range(n - 1, n - 5, -1)) if o.control is not None],
    "q4_hi_first30": qft_stages(n, range(n - 1, n - 5, -1))[:30],
    "q4_mid": qft_stages(n, range(17, 13, -1)),
    "q4_lo": qft_stages(n, range(9, 5, -1)),
    "q4_lo_noH": [o for o in qft_stages(n, range(9, 5, -1)) if o.control is not None],
    "4H_hi": [sv.GateOp(sv.hadamard(), t) for t in range(n - 1, n - 5, -1)],
    "4H_lo": [sv.GateOp(sv.hadamard(), t) for t in range(9, 5, -1)],
    "phase_hi_ctl_hi_30": [sv.GateOp(sv.phase_r(3), n - 1, c) for c in range(10, 25)] * 2,
    "phase_hi_ctl_lanes_30": [sv.GateOp(sv.phase_r(3), n - 1, c) for c in range(0, 5)] * 6,
    "phase_hi_unctl_30": [sv.GateOp(sv.phase_r(3), n - 1)] * 30,
    "phase_hi_ctl_hi_110": [sv.GateOp(sv.phase_r(3), n - 1, c) for c in range(10, 25)] * 7 + [
        sv.GateOp(sv.phase_r(3), n - 1, 12)] * 5,
    "phase_hi_unctl_60": [sv.GateOp(sv.phase_r(3), n - 1)] * 60,
    "phase_hi_unctl_110": [sv.GateOp(sv.phase_r(3), n - 1)] * 110,
    "phase_4slots_ctl_hi_110": [sv.GateOp(sv.phase_r(3), n - 1 - (i % 4), 10 + (i % 15)) for i in range(110)],
    "phase_ctl_one_hi_110": [sv.GateOp(sv.phase_r(3), n - 1, 15)] * 110,
    "phase_ctl_two_hi_110": [sv.GateOp(sv.phase_r(3), n - 1, 15 + (i % 2)) for i in range(110)],
    "phase_ctl_8bits_hi_110": [sv.GateOp(sv.phase_r(3), n - 1, 10 + (i % 8)) for i in range(110)],
    "phase_ctl_blocks_hi_110": [sv.GateOp(sv.phase_r(3), n - 1, 10 + i // 10) for i in range(110)],
    "general_hi_30": [sv.GateOp(sv.random_unitary(np.random.default_rng(i)), n - 1 - (i % 4)) for i in range(30)],
}
res = {"n": n}
for k, ops in cases.items():
    res[k] = {"gates": len(ops), "ms": timed(stage(ops), reps)}
print(json.dumps(res))
