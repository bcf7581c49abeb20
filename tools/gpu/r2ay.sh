mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -m gpu -q -x > gpurun_out/r2ay_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2ay_pytest.log
GROUPS=5 CONCS=3 timeout 300 python tools/sweep_ab.py > gpurun_out/r2ay_ab.log 2>&1
tail -3 gpurun_out/r2ay_pytest.log; cat gpurun_out/r2ay_ab.log
