mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_mstage.py -x -q > gpurun_out/ms_tests.log 2>&1; tail -15 gpurun_out/ms_tests.log
