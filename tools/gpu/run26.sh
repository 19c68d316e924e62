mkdir -p gpurun_out
O=gpurun_out/ms_stagger.txt
: > $O
for v in 0 20000000 12000 40000; do echo "== SVB_MS_STAGGER=$v" >> $O; SVB_MS_STAGGER=$v timeout 300 python tools/qft_breakdown.py 30 12 >> $O 2>&1; done
cat $O
