mkdir -p gpurun_out
cat > /tmp/small_sweep.py <<'PY'
import sys, os
sys.path.insert(0, ".")
import torch
from paper_1912_07133_b200 import _lib, detect, filters, synth
cat = filters.catalog()
n = int(sys.argv[1])
x = torch.from_numpy(synth.config3_frame(n)).cuda()
for grp in (5, 3, 1):
    detect.SWEEP_GROUP = grp
    stg = [detect.make_stage(cat[nm]) for nm in ["rp2", "rp4", "rp8", "rp16", "rp32"]]
    outs = [(torch.empty((1 << 12, 2), dtype=torch.int32, device="cuda"), torch.empty(1 << 12, device="cuda"), torch.empty(2, dtype=torch.int64, device="cuda")) for _ in stg]
    detect._sweep_launch(x, _lib.VMF_F32, stg, 0.5, None, 1 << 12, outs, conc=1)
    torch.cuda.synchronize()
    print("n", n, "grp", grp, "ok", flush=True)
PY
for v in ""; do echo "== $v"; CUDA_LAUNCH_BLOCKING=1 timeout 120 python /tmp/small_sweep.py 4096 2>&1 | tail -2; VMF_ROWS_G2=1 CUDA_LAUNCH_BLOCKING=1 timeout 120 python /tmp/small_sweep.py 4096 2>&1 | tail -2; done
