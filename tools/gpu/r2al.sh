mkdir -p gpurun_out
timeout 300 python tools/diag/tl_firtc.py > gpurun_out/r2al.log 2>&1
cat gpurun_out/r2al.log
