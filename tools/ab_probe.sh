#!/bin/bash
# A/B the libsvb200 variants in build/variants/ (tools/build_variant.py) with tools/stage_probe.py and
# tools/time_fused.py (run under gpurun): bash tools/ab_probe.sh "name1 name2 ..."
O=gpurun_out/ab; mkdir -p $O
cp paper_1601_07195_b200/libsvb200.so /tmp/orig.so
for v in $1; do
  cp build/variants/$v/libsvb200.so paper_1601_07195_b200/libsvb200.so
  echo "== $v" >> $O/probe.txt
  python tools/stage_probe.py 30 3 >> $O/probe.txt 2>&1
  python tools/time_fused.py 30 3 >> $O/probe.txt 2>&1
done
cp /tmp/orig.so paper_1601_07195_b200/libsvb200.so
