"""Loopback timing of the global-qubit kernels (run under gpurun): two rank slices of 2^m
amplitudes on ONE GPU, so "remote" traffic is local HBM traffic -- a kernel-level ceiling,
not an NVLink number.

    python tools/time_global.py [m] [reps]

Per kernel: ms (median, CUDA events) and HBM GB/s of its algorithmic bytes.
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1601_07195_b200 as sv  # noqa: E402
from paper_1601_07195_b200 import _lib  # noqa: E402
from paper_1601_07195_b200.kernels import stream_handle  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 29
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
torch.cuda.set_device(0)
L = _lib.load()
a = sv.init_random_state(sv.Layout(m), seed=1).amps
b = sv.init_random_state(sv.Layout(m), seed=2).amps
signs = [torch.empty(_lib.diag_sign_bytes(m), dtype=torch.uint8, device="cuda") for _ in range(2)]
flags = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(2)]
h = sv.random_unitary(np.random.default_rng(0)).qbuf()
z = sv.phase_shift(0.3).qbuf()


def timed(fn):
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


st = stream_handle()
slice_b = 16 << m
res = {"m": m}
# one gate on the pairing bit: both sides' kernels (each half the pairs) = every element of both
# slices read and written once
t = timed(lambda: [_lib.check(L.sv_exchange(x.data_ptr(), y.data_ptr(), m, zr, -1, h, st))
                   for x, y, zr in ((a, b, 1), (b, a, 0))])
res["exchange"] = {"ms": round(t, 3), "hbm_gbs": round(4 * slice_b / t / 1e6, 1)}
t = timed(lambda: [_lib.check(L.sv_swap_global(x.data_ptr(), y.data_ptr(), m, zr, m - 3, st))
                   for x, y, zr in ((a, b, 1), (b, a, 0))])
res["swap_global"] = {"ms": round(t, 3), "hbm_gbs": round(2 * slice_b / t / 1e6, 1)}
t = timed(lambda: [_lib.check(L.sv_diag_global(x.data_ptr(), m, zr, -1, z, s.data_ptr(), f.data_ptr(), st))
                   for x, zr, s, f in ((a, 1, signs[0], flags[0]), (b, 0, signs[1], flags[1]))])
res["diag_global"] = {"ms": round(t, 3), "hbm_gbs": round(4 * slice_b / t / 1e6, 1)}
t = timed(lambda: [_lib.check(L.sv_diag_fix(x.data_ptr(), m, zr, -1, z, s.data_ptr(), f.data_ptr(), st))
                   for x, zr, s, f in ((a, 1, signs[1], flags[0]), (b, 0, signs[0], flags[1]))])
res["diag_fix_noop"] = {"ms": round(t, 4)}
t = timed(lambda: _lib.check(L.sv_apply_single(a.data_ptr(), m, m - 1, h, st)))
res["single_ref"] = {"ms": round(t, 3), "hbm_gbs": round(2 * slice_b / t / 1e6, 1)}
print(json.dumps(res))
