mkdir -p gpurun_out
GROUPS=5 CONCS=5 timeout 120 python tools/sweep_ab.py > gpurun_out/r2ch_ab.json 2>&1
timeout 120 python tools/sweep_timeline.py > gpurun_out/r2ch_tl.json 2>&1
timeout 900 python -m pytest tests/ -m gpu -q -x > gpurun_out/r2ch_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2ch_pytest.log
