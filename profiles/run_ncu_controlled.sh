#!/bin/bash
# ncu capture of the controlled-gate kernels (one GPU): (c, t) = (5, 17), (1, 17), (0, 17) at n = 28
# (tools/profile_controlled.py), the three DRAM regimes of sv_apply_controlled.
set -e
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
python tools/profile_controlled.py 28 > $OUT/ncu_ctl_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pairs|k_shfl" -c 3 -o $OUT/prof_controlled \
    python tools/profile_controlled.py 28 > $OUT/ncu_ctl.log 2>&1
