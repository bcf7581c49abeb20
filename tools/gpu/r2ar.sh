mkdir -p gpurun_out
timeout 300 python tools/diag/tl_firtc.py g32_k128 > gpurun_out/r2ar.log 2>&1
cat gpurun_out/r2ar.log
