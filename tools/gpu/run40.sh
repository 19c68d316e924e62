mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_tolerance.py -x -q > gpurun_out/tol_tests.log 2>&1; tail -5 gpurun_out/tol_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
