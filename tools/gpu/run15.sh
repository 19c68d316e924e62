mkdir -p gpurun_out
cp paper_1601_07195_b200/libsvb200.so /tmp/main.so
python -m pytest tests/test_gpu_bounds.py tests/test_gpu_tolerance.py -x -q > gpurun_out/t15.log 2>&1; tail -3 gpurun_out/t15.log
for v in main dlnopf; do
  if [ $v != main ]; then cp build/variants/$v/libsvb200.so paper_1601_07195_b200/libsvb200.so; fi
  echo "== $v"; python tools/time_tol.py 30 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['qft_tol_ms'], d['qft_tol_passes'])"
  cp /tmp/main.so paper_1601_07195_b200/libsvb200.so
done
