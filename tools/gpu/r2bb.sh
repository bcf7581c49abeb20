mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -m gpu -q -x > gpurun_out/r2bb_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2bb_pytest.log
tail -3 gpurun_out/r2bb_pytest.log
