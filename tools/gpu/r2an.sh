mkdir -p gpurun_out
CMD="python tools/diag/time_firtc.py g32_k128"
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:firtc_prep" -s 3 -c 1 -o gpurun_out/r2an_full $CMD > gpurun_out/r2an_ncu.log 2>&1
tail -2 gpurun_out/r2an_ncu.log
