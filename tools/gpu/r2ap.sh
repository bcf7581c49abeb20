mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -m gpu -q -x > gpurun_out/r2ap_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2ap_pytest.log
timeout 400 python bench.py > gpurun_out/r2ap_bench.json 2> gpurun_out/r2ap_bench.err
tail -5 gpurun_out/r2ap_pytest.log
