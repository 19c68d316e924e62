mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dstage -s 1 -c 1 -o gpurun_out/dstage2 python tools/time_tol.py 28 1 > gpurun_out/t7_ncu.log 2>&1; tail -2 gpurun_out/t7_ncu.log
