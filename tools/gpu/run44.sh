mkdir -p gpurun_out
OUT=gpurun_out
python bench.py > $OUT/r02_bench_default.json 2> $OUT/r02_bench_default.err; tail -1 $OUT/r02_bench_default.err
timeout 900 python bench.py --impl reference > $OUT/r02_bench_ref.json 2> $OUT/r02_bench_ref.err; tail -1 $OUT/r02_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/r02_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/r02_ncu_bench.log 2>&1; tail -c 300 $OUT/r02_ncu_bench.log
