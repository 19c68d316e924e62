#!/bin/bash
# A/B variants (tools/build_variant.py) on the QFT(30) pass plan and the random steps:
#   bash tools/ab_qft.sh "v1 v2 ..." [n]
O=gpurun_out/ab_qft.txt
mkdir -p gpurun_out
: > $O
cp paper_1601_07195_b200/libsvb200.so /tmp/orig.so.bak
for v in $1; do
  cp build/variants/$v/libsvb200.so paper_1601_07195_b200/libsvb200.so
  echo "== $v" >> $O
  timeout 300 python tools/qft_breakdown.py ${2:-30} 12 >> $O 2>&1
  timeout 300 python tools/time_stagger.py ${2:-30} 5 >> $O 2>&1
done
cp /tmp/orig.so.bak paper_1601_07195_b200/libsvb200.so
cat $O
