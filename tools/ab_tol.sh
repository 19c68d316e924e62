#!/bin/bash
# A/B variants (tools/build_variant.py) on the QFT tolerance plan: bash tools/ab_tol.sh "v1 v2 ..." [n]
O=gpurun_out/ab_tol.txt
mkdir -p gpurun_out
: > $O
cp paper_1601_07195_b200/libsvb200.so /tmp/orig.so.bak
for v in $1; do
  cp build/variants/$v/libsvb200.so paper_1601_07195_b200/libsvb200.so
  echo "== $v" >> $O
  timeout 300 python tools/time_tol.py ${2:-30} 5 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print({k:v for k,v in d.items() if 'qft_tol' in k})" >> $O
done
cp /tmp/orig.so.bak paper_1601_07195_b200/libsvb200.so
cat $O
