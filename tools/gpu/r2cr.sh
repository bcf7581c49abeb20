mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2cr_bench.json 2> gpurun_out/r2cr_bench.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra"
$CMD > gpurun_out/r2cr_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r2cr_launches.csv $CMD > gpurun_out/r2cr_ncu_list.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none \
    -k "regex:sweep_rows|sweep_border|colcarry32v|colscan32|colapply32v|colfinal" -c 6 -o gpurun_out/r2cr_iir_full \
    $CMD > gpurun_out/r2cr_ncu_iir.log 2>&1
ls -la gpurun_out/ | grep r2cr
