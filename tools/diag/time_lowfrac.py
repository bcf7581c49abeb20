"""Per-kernel device times of one IIR scale at frac 0.5 and 0.05 (profile events)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1912_07133_b200 import _lib, detect, filters, synth

c = filters.catalog()
x = torch.from_numpy(synth.config3_frame(4096)).cuda()
for frac in (0.5, 0.05):
    for _ in range(3):
        d = detect.blur_laplacian_detect(x, c["rp4"], frac=frac)
    torch.cuda.synchronize()
    prof = {}
    for _ in range(5):
        _lib.profile_begin()
        d = detect.blur_laplacian_detect(x, c["rp4"], frac=frac)
        torch.cuda.synchronize()
        _lib.profile_stop()
        for k, (t, n) in _lib.profile_read().items():
            t0, n0 = prof.get(k, (0.0, 0)); prof[k] = (t0 + t, n0 + n)
    print(frac, d.count, {k: round(1e3 * t / 5, 1) for k, (t, n) in prof.items()}, flush=True)
