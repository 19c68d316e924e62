#!/bin/bash
# ncu captures of the fused kernels (multi-target stage pass, register tile) and the QFT pass-plan
# launch list -- one GPU.  Second round of tools/profile_kernels.py: k_tile launches 2 (random run)
# and 3 (QFT tail), k_mstage launch 8 (first QFT pass: 81 gates on qubits 25..27).
set -e
OUT=${OUT:-gpurun_out}
CMD="python tools/profile_kernels.py 28"
$CMD > $OUT/ncu_fused_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_fused.csv $CMD > $OUT/ncu_fl.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_mstage -s 8 -c 1 -o $OUT/prof_mstage $CMD > $OUT/ncu_mstage.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tile -s 2 -c 2 -o $OUT/prof_tile $CMD > $OUT/ncu_tile.log 2>&1
