mkdir -p gpurun_out
python tools/diag/diag_col32.py > gpurun_out/r2c_diag.log 2>&1
python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/r2c_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2c_pytest.log
python bench.py --no-extra --no-cpu-baseline > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
tail -5 gpurun_out/r2c_pytest.log
