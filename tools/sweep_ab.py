"""A/B timer of the 5-scale sweep (bench step) under env settings:
python tools/sweep_ab.py  -> prints ms per step (graph replay, L2 flushed)."""
import os, sys, json
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
res = {}
for grp in [int(v) for v in os.environ.get("GROUPS", "5,3,2,1").split(",")]:
    for conc in [int(v) for v in os.environ.get("CONCS", "3").split(",")]:
        detect.SWEEP_GROUP = grp
        step = lambda: detect._sweep_launch(x, _lib.VMF_F32, stg, 0.5, None, 1 << 18, outs, conc=conc)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        g.replay(); torch.cuda.synchronize()
        tot = 0.0
        for _ in range(20):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); g.replay(); b.record(); b.synchronize()
            tot += a.elapsed_time(b)
        res[f"grp{grp}_conc{conc}"] = round(tot / 20, 4)
        del g
        if os.environ.get("EAGER"):  # the same step launched eagerly (no graph)
            tot = 0.0
            for _ in range(20):
                flush.zero_()
                a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
                a.record(); step(); b.record(); b.synchronize()
                tot += a.elapsed_time(b)
            res[f"eager_grp{grp}_conc{conc}"] = round(tot / 20, 4)
print(json.dumps(res))
