mkdir -p gpurun_out
set -x
python -m pytest tests/test_gpu_tolerance.py tests/test_gpu_large.py -x -q --durations=15 > gpurun_out/t2_new.log 2>&1; tail -30 gpurun_out/t2_new.log
python bench.py > gpurun_out/b2_default.json 2> gpurun_out/b2_default.err; tail -3 gpurun_out/b2_default.err
SVB_SHARE_DEVICE=1 timeout 600 python bench.py --gpus 2 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/b2_share2.json 2> gpurun_out/b2_share2.err; tail -5 gpurun_out/b2_share2.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/b2_ref.json 2> gpurun_out/b2_ref.err; tail -3 gpurun_out/b2_ref.err
python -m pytest tests -m gpu -x -q > gpurun_out/t2_all.log 2>&1; tail -5 gpurun_out/t2_all.log
