mkdir -p gpurun_out
SVB_SHARE_DEVICE=1 timeout 1200 python bench.py --gpus 2 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --qubits 29 > gpurun_out/b19_share2.json 2> gpurun_out/b19_share2.err; echo rc=$?; tail -5 gpurun_out/b19_share2.err
python -c "import json; d=json.loads(open('gpurun_out/b19_share2.json').read()); print({k:d.get(k) for k in ('value','n_gpus','gpu_launches')}); print(d.get('planes')); print(d.get('nvlink')); print({k:(v['ms_per_step'],v.get('nvlink')) for k,v in d.get('secondary',{}).items()}); print(d['self_check'])"
