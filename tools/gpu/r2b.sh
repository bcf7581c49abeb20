mkdir -p gpurun_out
python tools/diag/diag_rp32.py rp32 rp16 rp4 bw48 > gpurun_out/r2b_diag.log 2>&1
python -m pytest tests -m gpu -q --durations=20 > gpurun_out/r2b_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2b_pytest.log
tail -30 gpurun_out/r2b_pytest.log
