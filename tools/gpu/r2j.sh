mkdir -p gpurun_out
timeout 300 python tools/diag/diag_col32.py > gpurun_out/r2j_diag.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/r2j_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2j_pytest.log
timeout 300 python bench.py --no-extra --no-cpu-baseline > gpurun_out/r2j_bench.json 2> gpurun_out/r2j_bench.err
tail -5 gpurun_out/r2j_pytest.log
