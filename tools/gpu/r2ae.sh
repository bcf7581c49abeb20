mkdir -p gpurun_out
timeout 300 python tools/diag/time_firtc.py > gpurun_out/r2ae.log 2>&1
CMD="python tools/diag/time_firtc.py"
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:firtc" -c 8 -o gpurun_out/r2ae_full $CMD > gpurun_out/r2ae_ncu.log 2>&1
cat gpurun_out/r2ae.log
