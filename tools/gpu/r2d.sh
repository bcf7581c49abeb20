mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extra"
$CMD > gpurun_out/r2d_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none \
    -k "regex:colcarry32|colscan32|colapply32|rowpass_tma" -c 4 -o gpurun_out/r2d_full \
    $CMD > gpurun_out/r2d_ncu.log 2>&1
tail -3 gpurun_out/r2d_ncu.log
