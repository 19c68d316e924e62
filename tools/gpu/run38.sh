mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_mstage.py tests/test_gpu_passes.py -x -q > gpurun_out/ms_tests.log 2>&1; tail -4 gpurun_out/ms_tests.log
timeout 300 python tools/qft_breakdown.py 30 12 > gpurun_out/qft_breakdown.txt 2>&1; cat gpurun_out/qft_breakdown.txt
