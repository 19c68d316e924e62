mkdir -p gpurun_out
OUT=gpurun_out
T=/tmp/ncu_caps; mkdir -p $T
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_tol26.csv python tools/profile_kernels.py 26 qft_tol > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_xstage2 -s 3 -c 1 -f -o $T/prof_xstage2 \
    python tools/profile_kernels.py 28 qft_tol > $OUT/ncu_xstage2.log 2>&1; tail -1 $OUT/ncu_xstage2.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dlow -s 1 -c 1 -f -o $T/prof_dlow \
    python tools/profile_kernels.py 26 qft_tol > $OUT/ncu_dlow.log 2>&1; tail -1 $OUT/ncu_dlow.log
for k in prof_xstage2 prof_dlow; do
  ncu -i $T/$k.ncu-rep --page raw --csv > $OUT/$k.raw.csv 2>/dev/null
  ncu -i $T/$k.ncu-rep --page source --csv --print-source sass > $OUT/$k.sass.csv 2>/dev/null
  gzip -f $OUT/$k.sass.csv
done
ls -la $OUT | grep prof_
