"""A/B of the end-to-end stream (bench.py's e2e): 64 pinned 4096^2 frames
through detect.stream_sweep, wall clock, 3 repetitions per setting.
SCALE_STREAMS=3,5 python tools/e2e_ab.py"""
import json
import os
import sys
import time

sys.path.insert(0, ".")
import torch

from paper_1912_07133_b200 import detect, filters, synth

cat = filters.catalog()
frame = synth.config3_frame(4096)
host = torch.from_numpy(frame).pin_memory()
stages = [cat[n] for n in ["rp2", "rp4", "rp8", "rp16", "rp32"]]
n = 64
res = {}
for ss in [int(v) for v in os.environ.get("SCALE_STREAMS", "3,5").split(",")]:
    detect.SWEEP_SCALE_STREAMS = ss
    detect.stream_sweep([host] * n, stages)
    torch.cuda.synchronize()
    best = []
    for _ in range(3):
        t0 = time.perf_counter()
        detect.stream_sweep([host] * n, stages)
        torch.cuda.synchronize()
        best.append(time.perf_counter() - t0)
    mpx = frame.size / 1e6
    res[f"streams{ss}"] = [round(mpx * 5 * n / t, 1) for t in best]
print(json.dumps(res))
