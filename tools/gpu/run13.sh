mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_dlow|k_dstage" -c 2 -o gpurun_out/dlow2 python tools/time_tol.py 28 1 > gpurun_out/t13_ncu.log 2>&1; tail -1 gpurun_out/t13_ncu.log
