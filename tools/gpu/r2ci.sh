mkdir -p gpurun_out
GROUPS=5 CONCS=5 timeout 120 python tools/sweep_ab.py > gpurun_out/r2ci_ab.json 2>&1
timeout 120 python tools/sweep_timeline.py > gpurun_out/r2ci_tl.json 2>&1
timeout 300 python bench.py --no-extra --no-cpu-baseline --steps 20 > gpurun_out/r2ci_bench.json 2>gpurun_out/r2ci_bench.err
