mkdir -p gpurun_out
cat > /tmp/small_sweep.py <<'PY'
import sys, os
sys.path.insert(0, ".")
import torch
from paper_1912_07133_b200 import _lib, detect, filters, synth
cat = filters.catalog()
x = torch.from_numpy(synth.config3_frame(512)).cuda()
for grp in (5, 3, 2, 1):
    detect.SWEEP_GROUP = grp
    stg = [detect.make_stage(cat[n]) for n in ["rp2", "rp4", "rp8", "rp16", "rp32"]]
    outs = [(torch.empty((1 << 12, 2), dtype=torch.int32, device="cuda"), torch.empty(1 << 12, device="cuda"), torch.empty(2, dtype=torch.int64, device="cuda")) for _ in stg]
    detect._sweep_launch(x, _lib.VMF_F32, stg, 0.5, None, 1 << 12, outs, conc=3)
    torch.cuda.synchronize()
    print("grp", grp, "ok", flush=True)
PY
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python /tmp/small_sweep.py > gpurun_out/r2au_san.log 2>&1
VMF_ROWS_G2=1 timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python /tmp/small_sweep.py > gpurun_out/r2au_san2.log 2>&1
GROUPS=5,3 CONCS=3 timeout 300 python tools/sweep_ab.py > gpurun_out/r2au_ab.log 2>&1
tail -15 gpurun_out/r2au_san.log; tail -8 gpurun_out/r2au_san2.log; cat gpurun_out/r2au_ab.log | tail -3
