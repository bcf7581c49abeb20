mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_config_sizes.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r2s_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2s_pytest.log
timeout 300 python bench.py --no-extra --no-cpu-baseline > gpurun_out/r2s_bench.json 2> gpurun_out/r2s_bench.err
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extra"
$CMD > gpurun_out/r2s_plain.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none \
    -k "regex:sweep_rows" -c 1 -o gpurun_out/r2s_full \
    $CMD > gpurun_out/r2s_ncu.log 2>&1
tail -3 gpurun_out/r2s_pytest.log
