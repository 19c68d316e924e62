mkdir -p gpurun_out
SVB_SHARE_DEVICE=1 timeout 900 python bench.py --gpus 2 --steps 2 --warmup 3 > gpurun_out/r02_bench_shared2_diag.json 2> gpurun_out/r02_bench_shared2_diag.err; echo rc=$?; tail -3 gpurun_out/r02_bench_shared2_diag.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/r02_bench_shared2_diag.json'))
print(d['n_gpus'], d['config']['n_qubits'], d['config']['global_qubits'], d['value'], d.get('nvlink',{}).keys() if d.get('nvlink') else None, d['self_check'])
for k,v in d.get('secondary',{}).items(): print(k, v['ms_per_step'], v['hbm_passes_per_step'])
PY
