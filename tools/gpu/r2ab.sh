mkdir -p gpurun_out
timeout 600 python tools/row_ablation.py > gpurun_out/r2ab_abl.log 2>&1
cat gpurun_out/r2ab_abl.log
