mkdir -p gpurun_out
GROUPS=5 CONCS=5 timeout 300 python tools/sweep_ab.py > gpurun_out/r2cd_ab_multi.json 2>&1
VMF_SCAN_SINGLE=1 GROUPS=5 CONCS=5 timeout 300 python tools/sweep_ab.py > gpurun_out/r2cd_ab_single.json 2>&1
timeout 900 python -m pytest tests/ -m gpu -q -x > gpurun_out/r2cd_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2cd_pytest.log
