mkdir -p gpurun_out
CMD="python tools/sweep_timeline.py"
REPS=1 $CMD > /dev/null 2>&1 && \
REPS=1 timeout 600 ncu --set full --import-source on --clock-control none \
    -k "regex:colapply32v|colcarry32v|colscan32|colfinal" -c 4 -o gpurun_out/r2dl_full $CMD > gpurun_out/r2dl_ncu.log 2>&1
echo "ncu exit $?"
