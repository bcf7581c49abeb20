mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extra"
$CMD > gpurun_out/r2ca_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none \
    -k "regex:colapply32v|colcarry32v|colscan32|sweep_rows" -c 4 -o gpurun_out/r2ca_full \
    $CMD > gpurun_out/r2ca_ncu.log 2>&1
echo "ncu exit $?"
