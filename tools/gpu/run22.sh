mkdir -p gpurun_out
O=gpurun_out/tile_probe2.jsonl
: > $O
timeout 300 python tools/tile_probe2.py 30 5 12 >> $O 2>&1
timeout 300 python tools/tile_probe2.py 30 5 11 >> $O 2>&1
SVB_TILE_STAGGER=20000000 timeout 300 python tools/tile_probe2.py 30 3 12 >> $O 2>&1
cat $O
