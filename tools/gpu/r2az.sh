mkdir -p gpurun_out
timeout 400 python bench.py > gpurun_out/r2az_bench.json 2> gpurun_out/r2az_bench.err
tail -2 gpurun_out/r2az_bench.err
