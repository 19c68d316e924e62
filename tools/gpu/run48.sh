mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/r02_gpu_tests.log 2>&1; tail -2 gpurun_out/r02_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; tail -1 gpurun_out/r02_smoke.log
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b.json 2> gpurun_out/b.err; echo bench rc=$?
python - <<'PY'
import json
d=json.load(open('gpurun_out/b.json'))
print(d['value'], d['self_check']['ok'])
for k,v in d.get('secondary',{}).items(): print(k, v['ms_per_step'], v['hbm_passes_per_step'])
PY
