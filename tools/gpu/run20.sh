mkdir -p gpurun_out
S=$(date +%s)
python -m pytest tests -m gpu -q -x > gpurun_out/r02b_gpu_tests.log 2>&1; tail -3 gpurun_out/r02b_gpu_tests.log
echo "tests $(( $(date +%s) - S )) s"; S=$(date +%s)
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02b_smoke.log 2>&1; tail -1 gpurun_out/r02b_smoke.log
echo "smoke $(( $(date +%s) - S )) s"; S=$(date +%s)
python bench.py > gpurun_out/r02b_bench_default.json 2> gpurun_out/r02b_bench_default.err; tail -2 gpurun_out/r02b_bench_default.err
echo "bench $(( $(date +%s) - S )) s"; S=$(date +%s)
timeout 900 python bench.py --impl reference > gpurun_out/r02b_bench_ref.json 2> gpurun_out/r02b_bench_ref.err; tail -2 gpurun_out/r02b_bench_ref.err
echo "ref $(( $(date +%s) - S )) s"
