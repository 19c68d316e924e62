mkdir -p gpurun_out
python -m pytest tests/test_gpu_bounds.py tests/test_gpu_tolerance.py -x -q > gpurun_out/t14.log 2>&1; tail -3 gpurun_out/t14.log
python tools/time_tol.py 30 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['qft_tol_ms'], d['qft_tol_passes'])"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dlow -c 1 -o gpurun_out/dlow3 python tools/time_tol.py 28 1 > gpurun_out/t14_ncu.log 2>&1; tail -1 gpurun_out/t14_ncu.log
