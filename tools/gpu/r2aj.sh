mkdir -p gpurun_out
for v in "" build/abl/libtc1.so build/abl/libtc2.so build/abl/libtc3.so; do echo "== $v" >> gpurun_out/r2aj.log; VMF_LIB_PATH=$v timeout 300 python tools/diag/time_firtc.py >> gpurun_out/r2aj.log 2>&1; done
cat gpurun_out/r2aj.log
