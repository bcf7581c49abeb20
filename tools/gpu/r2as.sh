mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra"
$CMD > gpurun_out/r2as_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r2as_launches.csv $CMD > gpurun_out/r2as_ncu_list.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none \
    -k "regex:sweep_rows|sweep_border|colcarry32v|colscan32|colapply32v|colfinal" -c 6 -o gpurun_out/r2as_iir_full \
    $CMD > gpurun_out/r2as_ncu_iir.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none \
    -k "regex:firtc_mma|firtc_prep|firtc_nms" -s 3 -c 4 -o gpurun_out/r2as_fir_full \
    $CMD > gpurun_out/r2as_ncu_fir.log 2>&1
ls -la gpurun_out/ | grep r2as
