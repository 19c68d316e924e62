mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tolerance.py tests/test_gpu_bounds.py -x -q > gpurun_out/tol_tests.log 2>&1; tail -3 gpurun_out/tol_tests.log
timeout 300 python tools/time_tol.py 30 5 > gpurun_out/time_tol.json 2>&1; python - <<'PY'
import json
d=json.loads(open('gpurun_out/time_tol.json').read().strip().splitlines()[-1])
for k,v in d.items():
    if 'qft' in k or 'random25_tol' in k: print(k, v)
PY
cp build/variants/nosplit/libsvb200.so paper_1601_07195_b200/libsvb200.so
timeout 300 python tools/time_tol.py 30 5 > gpurun_out/time_tol_nosplit.json 2>&1; python - <<'PY'
import json
d=json.loads(open('gpurun_out/time_tol_nosplit.json').read().strip().splitlines()[-1])
for k,v in d.items():
    if 'qft_tol' in k: print('nosplit', k, v)
PY
