mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -m gpu -q -x > gpurun_out/r2cb_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2cb_pytest.log
tail -3 gpurun_out/r2cb_pytest.log
GROUPS=5 CONCS=3 timeout 300 python tools/sweep_ab.py > gpurun_out/r2cb_ab.json 2>&1
cat gpurun_out/r2cb_ab.json
timeout 300 python bench.py --no-extra --no-cpu-baseline > gpurun_out/r2cb_bench.json 2> gpurun_out/r2cb_bench.err
