mkdir -p gpurun_out
for i in 1 2; do
  GROUPS=5 CONCS=5 VMF_WALK_SEQ=1 timeout 200 python tools/sweep_ab.py >> gpurun_out/r2eb_ab.log 2>&1; echo "^seq" >> gpurun_out/r2eb_ab.log
  GROUPS=5 CONCS=5 timeout 200 python tools/sweep_ab.py >> gpurun_out/r2eb_ab.log 2>&1; echo "^pair" >> gpurun_out/r2eb_ab.log
done
timeout 900 python -m pytest tests/test_gpu_config_sizes.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r2eb_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2eb_pytest.log
timeout 300 python bench.py --no-extra --no-cpu-baseline > gpurun_out/r2eb_bench.json 2> gpurun_out/r2eb_bench.err
cat gpurun_out/r2eb_ab.log; tail -2 gpurun_out/r2eb_pytest.log
