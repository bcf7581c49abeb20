"""One fused scale (rp8 rows + columns + detection) on a 4096^2 synthetic
frame, run `reps` times -- a small target for ncu captures.

usage: python tools/prof_scale.py [stage] [reps] [size]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_07133_b200 import _lib, detect, filters, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "rp8"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
n = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
frame = synth.config3_frame(n)
x = torch.as_tensor(frame).cuda()
lap = torch.empty_like(x)
stg = detect.make_stage(filters.catalog()[name])
for _ in range(reps):
    detect._fused(x, _lib.VMF_F32, stg, stg, 1.0, 0.5, None, lap, 1 << 18, False)
torch.cuda.synchronize()
print("ok", name, reps, n)
