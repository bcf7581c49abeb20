mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -m gpu -q -x > gpurun_out/r2e3_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2e3_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e3_smoke.log 2>&1; echo "exit $?" >> gpurun_out/r2e3_smoke.log
timeout 900 python bench.py > gpurun_out/r2e3_bench.json 2> gpurun_out/r2e3_bench.err; echo "exit $?" >> gpurun_out/r2e3_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r2e3_ref.json 2> gpurun_out/r2e3_ref.err; echo "exit $?" >> gpurun_out/r2e3_ref.err
tail -3 gpurun_out/r2e3_pytest.log; tail -2 gpurun_out/r2e3_smoke.log; tail -1 gpurun_out/r2e3_bench.err; tail -1 gpurun_out/r2e3_ref.err
