mkdir -p gpurun_out
python -m pytest tests/test_gpu_tolerance.py tests/test_gpu_exchange.py -x -q > gpurun_out/t4.log 2>&1; tail -3 gpurun_out/t4.log
python tools/time_tol.py 30 5 > gpurun_out/t4_time.log 2>&1; cat gpurun_out/t4_time.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dstage -s 2 -c 1 -o gpurun_out/dstage python tools/time_tol.py 28 1 > gpurun_out/t4_ncu.log 2>&1; tail -2 gpurun_out/t4_ncu.log
