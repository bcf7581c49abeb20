mkdir -p gpurun_out
timeout 300 python tools/diag/diag_col32.py > gpurun_out/r2o_diag.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/r2o_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2o_pytest.log
timeout 300 python bench.py --no-extra --no-cpu-baseline > gpurun_out/r2o_bench.json 2> gpurun_out/r2o_bench.err
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extra"
$CMD > gpurun_out/r2o_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none \
    -k "regex:sweep_rows|sweep_border|colcarry32v|colscan32|colapply32v|colfinal" -c 10 -o gpurun_out/r2o_full \
    $CMD > gpurun_out/r2o_ncu.log 2>&1
tail -3 gpurun_out/r2o_pytest.log
