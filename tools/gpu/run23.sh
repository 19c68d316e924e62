mkdir -p gpurun_out
O=gpurun_out/qft_breakdown.txt
: > $O
for n in 30 26 22; do echo "== n=$n" >> $O; timeout 300 python tools/qft_breakdown.py $n 12 >> $O 2>&1; done
echo "== n=22 tile probe" >> $O
timeout 300 python tools/tile_probe2.py 22 5 12 >> $O 2>&1
cat $O
