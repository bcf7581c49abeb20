mkdir -p gpurun_out
for v in "" build/abl/libtc1.so build/abl/libtc4.so build/abl/libtc5.so; do echo "== $v" >> gpurun_out/r2aq.log; VMF_LIB_PATH=$v timeout 300 python tools/diag/time_firtc.py >> gpurun_out/r2aq.log 2>&1; done
cat gpurun_out/r2aq.log
