mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_config_sizes.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r2z_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2z_pytest.log
timeout 300 python bench.py --no-extra --no-cpu-baseline > gpurun_out/r2z_bench.json 2> gpurun_out/r2z_bench.err
tail -2 gpurun_out/r2z_pytest.log
