"""Per-scale FIR timing on the config-3 frame (4096^2): each Gaussian FIR
scale (rows + fused columns + finaliser) as one CUDA graph, L2 flushed, median
of `reps` replays.  A/B helper for the FIR kernels (run it under different
VMF_* environment settings).

usage: python tools/fir_ab.py [reps] [size]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_07133_b200 import _lib, detect, filters, synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 9
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
x = torch.as_tensor(synth.config3_frame(n)).cuda()
lap = torch.empty_like(x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
cat = filters.catalog()
out = {}
for name in ("g2_k8", "g4_k16", "g8_k32", "g16_k64", "g32_k128"):
    stg = detect.make_stage(cat[name])

    def one():
        detect._fused(x, _lib.VMF_F32, stg, stg, 1.0, 0.5, None, lap, 1 << 18, False)

    one()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        one()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    out[name] = round(ts[len(ts) // 2], 1)
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("VMF_")},
                  "us_per_scale": out}))
