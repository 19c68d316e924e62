mkdir -p gpurun_out
S=$(date +%s)
python -m pytest tests -m gpu -x -q > gpurun_out/r02d_gpu_tests.log 2>&1; tail -3 gpurun_out/r02d_gpu_tests.log
echo "tests $(( $(date +%s) - S )) s"; S=$(date +%s)
python bench.py > gpurun_out/r02d_bench_default.json 2> gpurun_out/r02d_bench_default.err; tail -2 gpurun_out/r02d_bench_default.err
echo "bench $(( $(date +%s) - S )) s"
python - <<'PY'
import json
d=json.load(open('gpurun_out/r02d_bench_default.json'))
print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['self_check'])
for k,v in d.get('secondary',{}).items(): print(k, v['ms_per_step'], v['hbm_passes_per_step'], v['roofline'].get('frac'), v['roofline'].get('kernel'))
PY
