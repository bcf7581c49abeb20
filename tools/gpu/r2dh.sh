mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:firtc_" -s 8 -c 4 -o gpurun_out/r2dh_full python tools/scratch/fir_one.py > gpurun_out/r2dh_ncu.log 2>&1
echo "ncu exit $?"
