"""globaltimer timeline of the sweep row pass (build/tl/libtl.so, built with
-DVMF_TIMELINE=1): per-CTA launch / start (after griddepcontrol.wait) / end,
and per-row phase stamps of CTAs 0..7 (0: row TMA landed, 1: carries + B1,
2: scans + B2, 3: walks + V stores).  python tools/row_timeline.py"""
import ctypes as C
import json
import os
import sys

import numpy as np

os.environ["VMF_LIB_PATH"] = os.path.abspath("build/tl/libtl.so")
sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1912_07133_b200 import _lib, detect, filters, synth  # noqa: E402

cat = filters.catalog()
x = torch.from_numpy(synth.config3_frame(4096)).cuda()
stg = [detect.make_stage(cat[n]) for n in ["rp2", "rp4", "rp8", "rp16", "rp32"]]
outs = [(torch.empty((1 << 18, 2), dtype=torch.int32, device="cuda"),
         torch.empty(1 << 18, dtype=torch.float32, device="cuda"),
         torch.empty(2, dtype=torch.int64, device="cuda")) for _ in stg]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
L = _lib.lib()
L.vmf_debug_timeline.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros(4096, np.uint64)
res = []
for it in range(4):
    flush.zero_()
    torch.cuda.synchronize()
    L.vmf_debug_timeline_reset()
    detect._sweep_launch(x, _lib.VMF_F32, stg, 0.5, None, 1 << 18, outs)
    torch.cuda.synchronize()
    L.vmf_debug_timeline(buf.ctypes.data, 4096)
    t = buf.astype(np.int64)
    grid = int((t[:1024] > 0).sum())
    launch, start, end = t[2048:2048 + grid], t[:grid], t[1024:1024 + grid]
    t0 = launch.min()
    rows = t[2560:2560 + 8 * 16 * 4].reshape(8, 16, 4)
    ph = []
    for b in range(8):
        r = rows[b]
        n = int((r[:, 3] > 0).sum())
        prev = np.concatenate([[start[b]], r[:n - 1, 3]])
        ph.append({"cta": b, "rows": n,
                   "tma_wait_us": round(float(np.mean(r[:n, 0] - prev)) / 1e3, 2),
                   "carry_b1_us": round(float(np.mean(r[:n, 1] - r[:n, 0])) / 1e3, 2),
                   "scan_b2_us": round(float(np.mean(r[:n, 2] - r[:n, 1])) / 1e3, 2),
                   "walk_store_us": round(float(np.mean(r[:n, 3] - r[:n, 2])) / 1e3, 2)})
    res.append({"grid": grid, "span_us": round((end.max() - t0) / 1e3, 1),
                "start_after_launch_us": [round(float(np.percentile(start - t0, q)) / 1e3, 1) for q in (0, 50, 100)],
                "end_us_pct": [round(float(np.percentile(end - t0, q)) / 1e3, 1) for q in (0, 10, 50, 90, 100)],
                "edge_ctas": [[round((start[g] - t0) / 1e3, 1), round((end[g] - t0) / 1e3, 1)] for g in range(grid - 5, grid)],
                "row_phases": ph})
for r in res[1:]:
    print(json.dumps(r))
