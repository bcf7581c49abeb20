mkdir -p gpurun_out
GROUPS=5 CONCS=5 timeout 120 python tools/sweep_ab.py > gpurun_out/r2cu_ab.json 2>&1
VMF_NO_ROWT=1 GROUPS=5 CONCS=5 timeout 120 python tools/sweep_ab.py > gpurun_out/r2cu_ab_old.json 2>&1
timeout 120 python tools/sweep_timeline.py > gpurun_out/r2cu_tl.json 2>&1
timeout 600 python -m pytest tests/test_gpu_config_sizes.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r2cu_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2cu_pytest.log
