#!/bin/bash
# A/B the variants built by tools/build_variant.py (run under gpurun):
#   bash tools/ab_variants.sh "name1 name2 ..." [n] [pytest selection]
# Each variant: swap the .so in, time the fused kernels (tools/time_fused.py), run the GPU parity tests.
O=gpurun_out/ab
mkdir -p $O
cp paper_1601_07195_b200/libsvb200.so $O/orig.so.bak
for v in $1; do
  cp build/variants/$v/libsvb200.so paper_1601_07195_b200/libsvb200.so
  echo "== $v" >> $O/times.txt
  timeout 300 python tools/time_fused.py ${2:-30} 5 >> $O/times.txt 2>&1
  if [ -n "$3" ]; then timeout 600 python -m pytest $3 -x -q > $O/pytest_$v.log 2>&1; echo "$v pytest rc=$?" >> $O/times.txt; fi
done
cp $O/orig.so.bak paper_1601_07195_b200/libsvb200.so
rm $O/orig.so.bak
