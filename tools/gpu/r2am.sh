mkdir -p gpurun_out
timeout 900 python tools/diag/diag_firtc.py > gpurun_out/r2am_firtc.log 2>&1; echo "exit $?" >> gpurun_out/r2am_firtc.log
timeout 300 python tools/diag/time_firtc.py > gpurun_out/r2am_time.log 2>&1
CMD="python tools/diag/time_firtc.py"
cat gpurun_out/r2am_firtc.log | tail -11; cat gpurun_out/r2am_time.log
