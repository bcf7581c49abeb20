mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -m gpu -q > gpurun_out/r2e1_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2e1_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e1_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r2e1_bench.json 2> gpurun_out/r2e1_bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2e1_ref.json 2> gpurun_out/r2e1_ref.err
timeout 200 python tools/sweep_timeline.py > gpurun_out/r2e1_tl.json 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra"
$CMD > gpurun_out/r2e1_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r2e1_launches.csv $CMD > gpurun_out/r2e1_ncu_list.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none \
    -k "regex:sweep_rows|sweep_border|colcarry32v|colscan32|colapply32v|colfinal" -c 6 -o gpurun_out/r2e1_iir_full \
    $CMD > gpurun_out/r2e1_ncu_iir.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:firtc_" -s 8 -c 4 -o gpurun_out/r2e1_fir_full python tools/fir_one.py > gpurun_out/r2e1_ncu_fir.log 2>&1
ls -la gpurun_out/ | grep r2e1
