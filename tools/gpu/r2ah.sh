mkdir -p gpurun_out
timeout 900 python tools/diag/diag_firtc.py > gpurun_out/r2ah_firtc.log 2>&1; echo "exit $?" >> gpurun_out/r2ah_firtc.log
timeout 300 python tools/diag/time_firtc.py > gpurun_out/r2ah_time.log 2>&1
CMD="python tools/diag/time_firtc.py"
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:firtc" -c 3 -o gpurun_out/r2ah_full $CMD > gpurun_out/r2ah_ncu.log 2>&1
cat gpurun_out/r2ah_firtc.log | tail -11; cat gpurun_out/r2ah_time.log
