mkdir -p gpurun_out
VMF_ROWS_G2=1 timeout 900 python -m pytest tests/test_gpu_config_sizes.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r2at_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2at_pytest.log
GROUPS=5 CONCS=3 timeout 300 python tools/sweep_ab.py > gpurun_out/r2at_ab.log 2>&1
VMF_ROWS_G2=1 GROUPS=5 CONCS=3 timeout 300 python tools/sweep_ab.py >> gpurun_out/r2at_ab.log 2>&1
VMF_ROWS_G2=1 timeout 300 python tools/row_ablation.py > gpurun_out/r2at_abl.log 2>&1
tail -3 gpurun_out/r2at_pytest.log; cat gpurun_out/r2at_ab.log gpurun_out/r2at_abl.log
