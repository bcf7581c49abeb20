mkdir -p gpurun_out
GROUPS=5,3,2,1 CONCS=2,3,4 timeout 600 python tools/sweep_ab.py > gpurun_out/r2r_ab.log 2>&1
cat gpurun_out/r2r_ab.log | tail -3
