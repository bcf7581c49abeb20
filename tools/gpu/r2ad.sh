mkdir -p gpurun_out
timeout 900 python tools/diag/diag_firtc.py > gpurun_out/r2ad_firtc.log 2>&1; echo "exit $?" >> gpurun_out/r2ad_firtc.log
cat gpurun_out/r2ad_firtc.log | tail -15
