mkdir -p gpurun_out
CMD="python tools/diag/time_firtc.py"
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:firtc" -c 12 -o gpurun_out/r2ak_full $CMD > gpurun_out/r2ak_ncu.log 2>&1
tail -2 gpurun_out/r2ak_ncu.log
