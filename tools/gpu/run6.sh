mkdir -p gpurun_out
cp paper_1601_07195_b200/libsvb200.so /tmp/main.so
python -m pytest tests/test_gpu_mstage.py tests/test_gpu_passes.py tests/test_gpu_tolerance.py -x -q > gpurun_out/t6.log 2>&1; tail -3 gpurun_out/t6.log
for v in main nopipe; do
  if [ $v != main ]; then cp build/variants/$v/libsvb200.so paper_1601_07195_b200/libsvb200.so; fi
  echo "== $v"; python tools/time_tol.py 30 5
  cp /tmp/main.so paper_1601_07195_b200/libsvb200.so
done > gpurun_out/t6_time.log 2>&1
cat gpurun_out/t6_time.log | cut -c1-700
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_dstage|k_mstage_pipe" -s 4 -c 2 -o gpurun_out/pipe python tools/time_tol.py 28 1 > gpurun_out/t6_ncu.log 2>&1; tail -2 gpurun_out/t6_ncu.log
