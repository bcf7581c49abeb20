"""Per-kernel device times of one tensor-core FIR scale (profile events)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1912_07133_b200 import _lib, detect, filters, synth

c = filters.catalog()
x = torch.from_numpy(synth.config3_frame(4096)).cuda()
for name in ["g2_k8", "g8_k32", "g32_k128"]:
    f = c[name]
    for _ in range(3):
        detect.blur_laplacian_detect(x, f, frac=0.5)
    torch.cuda.synchronize()
    prof = {}
    for _ in range(5):
        _lib.profile_begin()
        detect.blur_laplacian_detect(x, f, frac=0.5)
        torch.cuda.synchronize()
        _lib.profile_stop()
        for k, (t, n) in _lib.profile_read().items():
            t0, n0 = prof.get(k, (0.0, 0)); prof[k] = (t0 + t, n0 + n)
    print(name, {k: round(1e3 * t / 5, 1) for k, (t, n) in prof.items()}, "us per call", flush=True)
