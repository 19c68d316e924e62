mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_mstage.py tests/test_gpu_passes.py tests/test_gpu_configs.py tests/test_gpu_properties.py tests/test_gpu_bounds.py -x -q > gpurun_out/ms_tests.log 2>&1; tail -12 gpurun_out/ms_tests.log
python - <<'PY'
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1601_07195_b200 as sv
from tools.time_fused import timed
n = 30
st = sv.init_random_state(sv.Layout(n), seed=1)
for inv in (False, True):
    circ = sv.build_qft(n)
    if inv: circ = circ.inverse()
    plan = sv.plan_passes(circ.gates, n, 12, exact=True)
    ts = [(p.kind, len(p.gates), round(timed(lambda p=p: sv.execute_pass(st, p, tile=12), 3), 2)) for p in plan]
    print(n, 'inverse' if inv else 'forward', round(sum(t[2] for t in ts), 2), ts)
PY
