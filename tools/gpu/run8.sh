mkdir -p gpurun_out
cp paper_1601_07195_b200/libsvb200.so /tmp/main.so
for v in msp3; do
  cp build/variants/$v/libsvb200.so paper_1601_07195_b200/libsvb200.so
  echo "== $v"; python tools/time_tol.py 30 3 | cut -c1-400
  cp /tmp/main.so paper_1601_07195_b200/libsvb200.so
done > gpurun_out/t8_time.log 2>&1
cat gpurun_out/t8_time.log
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"k_pairs|k_shfl" -c 5 --csv python tools/profile_controlled.py 28 > gpurun_out/t8_ctl.csv 2>&1; tail -32 gpurun_out/t8_ctl.csv | cut -c1-250
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py tests/test_gpu_passes.py -x -q -k "golden or n5 or small or 12 or 10" > gpurun_out/t8_memcheck.log 2>&1; echo memcheck rc=$?; tail -5 gpurun_out/t8_memcheck.log
