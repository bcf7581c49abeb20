mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_firtc.py -m gpu -q -x > gpurun_out/r2ao.log 2>&1; echo "exit $?" >> gpurun_out/r2ao.log
tail -30 gpurun_out/r2ao.log
