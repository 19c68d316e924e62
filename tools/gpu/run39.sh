mkdir -p gpurun_out
O=gpurun_out/tol_sizes.txt
: > $O
for n in 31 32 33; do
python - <<PY >> $O 2>&1
import sys, json
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1601_07195_b200 as sv
from tools.time_fused import timed
n=$n
st = sv.init_random_state(sv.Layout(n), seed=1)
circ = sv.build_qft(n)
for exact in (True, False):
    plan = sv.plan_passes(circ.gates, n, 12, exact=exact)
    print(n, 'exact' if exact else 'tol', [(p.kind, len(p.gates), round(timed(lambda p=p: sv.execute_pass(st, p, tile=12), 2), 2)) for p in plan])
PY
done
cat $O
