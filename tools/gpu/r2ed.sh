mkdir -p gpurun_out
for i in 1 2; do GROUPS=5 CONCS=5 timeout 200 python tools/sweep_ab.py >> gpurun_out/r2ed_ab.log 2>&1; done
REPS=1 timeout 200 python tools/sweep_timeline.py > gpurun_out/r2ed_tl.json 2>&1
timeout 900 python -m pytest tests/test_gpu_config_sizes.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r2ed_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2ed_pytest.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:sweep_border -c 3 --csv $CMD > gpurun_out/r2ed_border.csv 2>&1
