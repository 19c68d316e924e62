mkdir -p gpurun_out
OUT=gpurun_out
T=/tmp/ncu_caps; mkdir -p $T
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mstage -s 6 -c 1 -f -o $T/prof_mstage \
    python tools/profile_kernels.py 28 qft > $OUT/ncu_mstage.log 2>&1; tail -1 $OUT/ncu_mstage.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tile -s 3 -c 1 -f -o $T/prof_tile_random \
    python tools/profile_kernels.py 28 random > $OUT/ncu_tile_random.log 2>&1; tail -1 $OUT/ncu_tile_random.log
for k in prof_mstage prof_tile_random; do
  ncu -i $T/$k.ncu-rep --page raw --csv > $OUT/$k.raw.csv 2>/dev/null
  ncu -i $T/$k.ncu-rep --page source --csv --print-source sass > $OUT/$k.sass.csv 2>/dev/null
  gzip -f $OUT/$k.sass.csv
done
ls -la $OUT
