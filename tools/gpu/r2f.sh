mkdir -p gpurun_out
timeout 300 python tools/diag/diag_col32.py > gpurun_out/r2f_diag.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/r2f_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2f_pytest.log
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extra"
$CMD > gpurun_out/r2f_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none \
    -k "regex:rowlap|colcarry32|colscan32|colapply32|rowfix" -c 5 -o gpurun_out/r2f_full \
    $CMD > gpurun_out/r2f_ncu.log 2>&1
tail -5 gpurun_out/r2f_pytest.log
