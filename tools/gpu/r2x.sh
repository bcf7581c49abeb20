mkdir -p gpurun_out
timeout 600 python tools/row_ablation.py > gpurun_out/r2x_abl.log 2>&1
timeout 300 python tools/row_timeline.py > gpurun_out/r2x_tl.log 2>&1
timeout 900 python -m pytest tests/test_gpu_config_sizes.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r2x_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2x_pytest.log
cat gpurun_out/r2x_abl.log; tail -1 gpurun_out/r2x_tl.log; tail -2 gpurun_out/r2x_pytest.log
