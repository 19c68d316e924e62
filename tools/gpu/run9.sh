mkdir -p gpurun_out
python -m pytest tests/test_gpu_bounds.py tests/test_gpu_tolerance.py -x -q > gpurun_out/t9.log 2>&1; tail -15 gpurun_out/t9.log
python tools/time_tol.py 30 5 > gpurun_out/t9_time.log 2>&1; cut -c1-900 gpurun_out/t9_time.log
