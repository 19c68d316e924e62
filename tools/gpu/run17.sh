mkdir -p gpurun_out
python -m pytest tests/test_gpu_tolerance.py tests/test_gpu_bounds.py -x -q > gpurun_out/t17.log 2>&1; tail -3 gpurun_out/t17.log
python tools/time_tol.py 30 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['qft_tol_ms'], d['qft_tol_passes']); print(d['random25_tol_ms'], d['ctl30_tol_ms'])"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dstage2 -c 1 -o gpurun_out/dstage2 python tools/time_tol.py 28 1 > gpurun_out/t17_ncu.log 2>&1; tail -1 gpurun_out/t17_ncu.log
