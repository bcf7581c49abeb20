"""A small pass over every kernel family of the hot path (a quick GPU smoke of
all of them in a few seconds; compute-sanitizer is closed on this pool): the 5-scale IIR detect sweep in every scale
grouping, the scale-space rule, a tensor-core FIR scale and an fp64 FIR scale,
and the u16 stream front end.  512^2 frames by default (N=...)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np
import torch

from paper_1912_07133_b200 import _lib, detect, filters, synth

cat = filters.catalog()
n = int(os.environ.get("N", "512"))
x = torch.from_numpy(synth.config3_frame(n)).cuda()
iir = ["rp2", "rp4", "rp8", "rp16", "rp32"]
for grp in (5, 3, 1):
    detect.SWEEP_GROUP = grp
    stg = [detect.make_stage(cat[k]) for k in iir]
    outs = [(torch.empty((1 << 12, 2), dtype=torch.int32, device="cuda"),
             torch.empty(1 << 12, device="cuda"),
             torch.empty(2, dtype=torch.int64, device="cuda")) for _ in stg]
    detect._sweep_launch(x, _lib.VMF_F32, stg, 0.5, None, 1 << 12, outs, conc=3)
    torch.cuda.synchronize()
    print("iir sweep, group", grp, "ok", [int(o[2][0]) for o in outs], flush=True)
detect.SWEEP_GROUP = 5
d = detect.detect_sweep(x, [cat[k] for k in iir], frac=0.05)
print("detect_sweep frac 0.05:", [len(q.y) for q in d], flush=True)
d = detect.scale_space_detect(x, [cat[k] for k in iir], [2, 4, 8, 16, 32], frac=0.5)
print("scale space:", len(d.y), flush=True)
for k in ("g2_k8", "g8_k32"):
    q = detect.detect_sweep(x, [cat[k]], frac=0.5)
    print("fir", k, len(q[0].y), flush=True)
fr = synth.config4_stream(n_frames=3, size=n)
r = detect.stream_detect(np.ascontiguousarray(fr), cat["rp6"], frac=0.5)
print("stream:", [len(q.y) for q in r], flush=True)
