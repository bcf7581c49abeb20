mkdir -p gpurun_out
CMD="python tools/sweep_timeline.py"
REPS=1 $CMD > /dev/null 2>&1 && \
REPS=1 timeout 600 ncu --set full --import-source on --clock-control none \
    -k "regex:sweep_rows" -c 1 -o gpurun_out/r2cy_full $CMD > gpurun_out/r2cy_ncu.log 2>&1
echo "ncu exit $?"
