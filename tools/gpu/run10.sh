mkdir -p gpurun_out
python -m pytest tests/test_gpu_bounds.py tests/test_gpu_tolerance.py -x -q > gpurun_out/t10.log 2>&1; tail -3 gpurun_out/t10.log
python tools/time_tol.py 30 5 > gpurun_out/t10_time.log 2>&1; cut -c1-900 gpurun_out/t10_time.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dlow -c 1 -o gpurun_out/dlow python tools/time_tol.py 28 1 > gpurun_out/t10_ncu.log 2>&1; tail -1 gpurun_out/t10_ncu.log
