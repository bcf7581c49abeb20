mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_config_sizes.py tests/test_gpu_parity.py tests/test_gpu_sweep.py -m gpu -q -x > gpurun_out/r2aa_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2aa_pytest.log
timeout 300 python bench.py --no-extra --no-cpu-baseline > gpurun_out/r2aa_bench.json 2> gpurun_out/r2aa_bench.err
GROUPS=5 CONCS=3 timeout 300 python tools/sweep_ab.py > gpurun_out/r2aa_ab.log 2>&1
VMF_NO_WS=1 GROUPS=5 CONCS=3 timeout 300 python tools/sweep_ab.py >> gpurun_out/r2aa_ab.log 2>&1
tail -3 gpurun_out/r2aa_pytest.log; cat gpurun_out/r2aa_ab.log
