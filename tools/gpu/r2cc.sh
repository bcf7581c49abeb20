mkdir -p gpurun_out
for pr in 0 1; do
  if [ $pr = 1 ]; then export VMF_SWEEP_PRIO=1; fi
  GROUPS=5 CONCS=3,4,5 timeout 300 python tools/sweep_ab.py > gpurun_out/r2cc_ab_p$pr.json 2>&1
  timeout 200 python tools/sweep_timeline.py > gpurun_out/r2cc_tl_p$pr.json 2>&1
done
python -c "import torch; print(torch.cuda.Stream.priority_range())" > gpurun_out/r2cc_prio.txt 2>&1
