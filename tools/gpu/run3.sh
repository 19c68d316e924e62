mkdir -p gpurun_out
cp paper_1601_07195_b200/libsvb200.so /tmp/main.so
python -m pytest tests/test_gpu_tolerance.py -x -q > gpurun_out/t3_tol.log 2>&1; tail -5 gpurun_out/t3_tol.log
for v in main ds2 ds4; do
  if [ $v != main ]; then cp build/variants/$v/libsvb200.so paper_1601_07195_b200/libsvb200.so; fi
  echo "== $v"; python tools/time_tol.py 30 5
  cp /tmp/main.so paper_1601_07195_b200/libsvb200.so
done > gpurun_out/t3_time.log 2>&1
tail -8 gpurun_out/t3_time.log
