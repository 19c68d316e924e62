mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_tolerance.py tests/test_gpu_bounds.py tests/test_gpu_mstage.py tests/test_gpu_passes.py -x -q > gpurun_out/tol_tests.log 2>&1; tail -12 gpurun_out/tol_tests.log
python - <<'PY'
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1601_07195_b200 as sv
from tools.time_fused import timed
for n, inv in ((30, False), (30, True), (31, False), (32, False)):
    st = sv.init_random_state(sv.Layout(n), seed=1)
    circ = sv.build_qft(n)
    if inv: circ = circ.inverse()
    plan = sv.plan_passes(circ.gates, n, 12, exact=False)
    ts = [(p.kind, len(p.gates), round(timed(lambda p=p: sv.execute_pass(st, p, tile=12), 3), 2)) for p in plan]
    print(n, 'inverse' if inv else 'forward', round(sum(t[2] for t in ts), 2), ts)
    del st; torch.cuda.empty_cache()
PY
