mkdir -p gpurun_out
O=gpurun_out/stagger.jsonl
: > $O
for v in 0 2000 5000 8000 12000 16000 24000; do
  SVB_TILE_STAGGER=$v SVB_MS_STAGGER=0 timeout 300 python tools/time_stagger.py 30 5 >> $O 2>&1
done
for v in 4000 8000 12000 16000 24000 36000; do
  SVB_TILE_STAGGER=0 SVB_MS_STAGGER=$v timeout 300 python tools/time_stagger.py 30 5 >> $O 2>&1
done
cat $O
