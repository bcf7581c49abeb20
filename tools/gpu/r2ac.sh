mkdir -p gpurun_out
timeout 60 ./tools/microbench/tc_tf32 > gpurun_out/tc_tf32.log 2>&1; echo "exit $?" >> gpurun_out/tc_tf32.log
cat gpurun_out/tc_tf32.log
