mkdir -p gpurun_out
cp paper_1601_07195_b200/libsvb200.so /tmp/main.so
python -m pytest tests/test_gpu_tolerance.py tests/test_gpu_exchange.py tests/test_gpu_shim.py tests/test_gpu_edges.py -x -q > gpurun_out/t5.log 2>&1; tail -3 gpurun_out/t5.log
for v in main ds3 ds1; do
  if [ $v != main ]; then cp build/variants/$v/libsvb200.so paper_1601_07195_b200/libsvb200.so; fi
  echo "== $v"; python tools/time_tol.py 30 5
  cp /tmp/main.so paper_1601_07195_b200/libsvb200.so
done > gpurun_out/t5_time.log 2>&1
cat gpurun_out/t5_time.log | cut -c1-600
