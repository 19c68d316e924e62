#!/bin/bash
# Profiling recipe (run under gpurun on ONE B200; see /opt/skills/guides/B200_PROFILING.md).
# 1) plain run must exit 0; 2) launch list; 3) --set full on the top kernels.
set -e
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
CMD="python bench.py --qubits 28 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > $OUT/ncu_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_shfl -s 60 -c 1 -o $OUT/prof_shfl $CMD > $OUT/ncu_full1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pairs -s 60 -c 1 -o $OUT/prof_pairs $CMD > $OUT/ncu_full2.log 2>&1
