"""Concurrent timeline of the bench step (the 5-scale IIR sweep on 3 streams):
event record nodes around every launch of ONE graph replay (L2 flushed
before), printed as (kernel, start, end) in us after the first launch.
python tools/sweep_timeline.py"""
import json
import os
import sys

sys.path.insert(0, ".")
import torch

from paper_1912_07133_b200 import _lib, detect, filters, synth

cat = filters.catalog()
x = torch.from_numpy(synth.config3_frame(4096)).cuda()
stg = [detect.make_stage(cat[n]) for n in ["rp2", "rp4", "rp8", "rp16", "rp32"]]
outs = [(torch.empty((1 << 18, 2), dtype=torch.int32, device="cuda"),
         torch.empty(1 << 18, dtype=torch.float32, device="cuda"),
         torch.empty(2, dtype=torch.int64, device="cuda")) for _ in stg]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
step = lambda: detect._sweep_launch(x, _lib.VMF_F32, stg, 0.5, None, 1 << 18, outs)
for _ in range(3):
    step()
torch.cuda.synchronize()
_lib.profile_begin()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
_lib.profile_stop()
res = []
for rep in range(int(os.environ.get("REPS", "3"))):
    flush.zero_()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    tl = _lib.profile_timeline()
    res.append([(k, round(a * 1e3, 1), round(b * 1e3, 1)) for k, a, b in tl])
for r in res:
    print(json.dumps({"span_us": max(b for _, _, b in r), "launches": r}))
