mkdir -p gpurun_out
GROUPS=5 CONCS=3 timeout 300 python tools/sweep_ab.py > gpurun_out/r2ax_ab.log 2>&1
VMF_ROWS_G2=1 GROUPS=5 CONCS=3 timeout 300 python tools/sweep_ab.py >> gpurun_out/r2ax_ab.log 2>&1
mv build/abl build/abl_off 2>/dev/null; mkdir -p build/abl
timeout 300 python tools/row_ablation.py > gpurun_out/r2ax_abl.log 2>&1
VMF_ROWS_G2=1 timeout 300 python tools/row_ablation.py >> gpurun_out/r2ax_abl.log 2>&1
cat gpurun_out/r2ax_ab.log gpurun_out/r2ax_abl.log
