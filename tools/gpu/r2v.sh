mkdir -p gpurun_out
timeout 300 python tools/row_timeline.py > gpurun_out/r2v_tl.log 2>&1
cat gpurun_out/r2v_tl.log | tail -3
