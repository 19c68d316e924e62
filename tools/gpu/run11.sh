mkdir -p gpurun_out
python -m pytest tests/test_gpu_bounds.py tests/test_gpu_tolerance.py -x -q > gpurun_out/t11.log 2>&1; tail -3 gpurun_out/t11.log
python tools/time_tol.py 30 5 > gpurun_out/t11_time.log 2>&1; cut -c1-700 gpurun_out/t11_time.log
