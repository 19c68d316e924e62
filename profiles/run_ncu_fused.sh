#!/bin/bash
# ncu captures of the fused kernels -- one GPU (tools/profile_kernels.py, second round of each):
#   k_mstage: first QFT(28) pass (four transform stages on qubits 24..27, 106 gates);
#   k_tile random: the first pass (9 gates) of the bench's config-4-shape step at n = 28 (gathered high qubits);
#   k_tile tile64: 64 random general gates on targets < 12 (FP64-bound extreme).
set -e
OUT=${OUT:-gpurun_out}
python tools/profile_kernels.py 28 > $OUT/ncu_fused_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_fused.csv \
    python tools/profile_kernels.py 28 > $OUT/ncu_fl.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_mstage -s 6 -c 1 -o $OUT/prof_mstage \
    python tools/profile_kernels.py 28 qft > $OUT/ncu_mstage.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tile -s 3 -c 1 -o $OUT/prof_tile_random \
    python tools/profile_kernels.py 28 random > $OUT/ncu_tile_random.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tile -s 1 -c 1 -o $OUT/prof_tile64 \
    python tools/profile_kernels.py 28 tile64 > $OUT/ncu_tile64.log 2>&1
