"""One 4096^2 detect call per FIR realisation (g8_k32: 65 taps, g32_k128: 257 taps),
three times each: the ncu target of the tensor-core FIR kernels."""
import sys; sys.path.insert(0, ".")
import torch
from paper_1912_07133_b200 import detect, filters, synth, _lib
cat = filters.catalog()
x = torch.from_numpy(synth.config3_frame(4096)).cuda()
for name in ["g8_k32", "g32_k128"]:
    stg = detect.make_stage(cat[name])
    for _ in range(3):
        detect._fused(x, _lib.VMF_F32, stg, stg, 1.0, 0.5, None, None, 1 << 18, False)
    torch.cuda.synchronize()
