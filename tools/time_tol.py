"""QFT(n) through the pass planner, exact vs tolerance mode (FusionConfig exact=False), with
per-pass CUDA-event times (run under gpurun).

    python tools/time_tol.py [n] [reps]
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1601_07195_b200 as sv  # noqa: E402


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


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    torch.cuda.set_device(0)
    st = sv.init_random_state(sv.Layout(n), seed=1)
    res = {"n": n}
    for name, circ in (("qft", sv.build_qft(n)),
                       ("random25", sv.random_circuit(n, 25, np.random.default_rng(1))),
                       ("ctl30", sv.random_circuit(n, 30, np.random.default_rng(1), controlled_fraction=1.0))):
        for exact in (True, False):
            fc = sv.FusionConfig(l_c=12, passes=True, exact=exact)
            key = f"{name}_{'exact' if exact else 'tol'}"
            res[key + "_ms"] = timed(lambda: sv.run_circuit(st, circ, fusion=fc), reps)
            plan = sv.plan_passes(circ.gates, n, 12, exact=exact)
            res[key + "_passes"] = [(p.kind, len(p.gates), round(timed(lambda p=p: sv.execute_pass(st, p, tile=12),
                                                                         reps), 3)) for p in plan]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
