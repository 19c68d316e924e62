mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02c_gpu_tests.log 2>&1; tail -3 gpurun_out/r02c_gpu_tests.log
timeout 300 python tools/time_fused.py 30 5 > gpurun_out/time_fused.json 2>&1; cat gpurun_out/time_fused.json
timeout 300 python tools/tile_probe2.py 30 5 12 >> gpurun_out/tile_probe2b.jsonl 2>&1; tail -1 gpurun_out/tile_probe2b.jsonl
