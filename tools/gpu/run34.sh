# Round-2 evidence run (one B200): tests, smoke, both bench arms, launch list, full captures.
mkdir -p gpurun_out
OUT=gpurun_out
T=/tmp/ncu_caps; mkdir -p $T
python -m pytest tests -m gpu -q > $OUT/r02_gpu_tests.log 2>&1; tail -2 $OUT/r02_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/r02_smoke.log 2>&1; tail -1 $OUT/r02_smoke.log
python bench.py > $OUT/r02_bench_default.json 2> $OUT/r02_bench_default.err; tail -1 $OUT/r02_bench_default.err
timeout 900 python bench.py --impl reference > $OUT/r02_bench_ref.json 2> $OUT/r02_bench_ref.err; tail -1 $OUT/r02_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/r02_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/r02_ncu_bench.log 2>&1; tail -1 $OUT/r02_ncu_bench.log
cap() {  # name regex skip n what
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -f -o $T/$1 \
      python tools/profile_kernels.py $4 $5 > $OUT/ncu_$1.log 2>&1
  ncu -i $T/$1.ncu-rep --page raw --csv > $OUT/$1.raw.csv 2>/dev/null
  ncu -i $T/$1.ncu-rep --page source --csv --print-source sass > $OUT/$1.sass.csv 2>/dev/null
  gzip -f $OUT/$1.sass.csv
  rm -f $T/$1.ncu-rep
}
cap prof_xstage2 k_xstage2 3 28 qft_tol
cap prof_dlow k_dlow 1 26 qft_tol
cap prof_mstage k_mstage 6 28 qft
cap prof_tile_random k_tile 3 28 random
ls -la $OUT | grep "prof_\|r02_"
