"""Tensor-core FIR path (vmf_firtc.cu) against the oracle: L error per kernel
/ shape, blob sets, and the time of one fused scale (against the fp64 FIR
path, VMF_NO_FIRTC)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O
from paper_1912_07133_b200 import _lib, detect, filters, synth
from tests.parity import compare_blobs

O.set_threads(O.max_threads())
c = filters.catalog()
cases = [("g2_k8", (512, 512)), ("g8_k32", (300, 516)), ("g4_k16", (257, 389)),
         ("g4_k16", (1000, 1032)), ("g16_k64", (1024, 1024)), ("g32_k128", (1024, 1024)),
         ("sg38.4", (1024, 1024)), ("g2_k8", (4096, 4096)), ("g32_k128", (4096, 4096))]
for name, (h, w) in cases:
    if (h, w) == (4096, 4096):
        x = synth.config3_frame(4096)
    else:
        rng = np.random.default_rng(h * 7 + w)
        x = (0.05 * rng.standard_normal((h, w))).astype(np.float32)
        yy, xx = np.ogrid[:h, :w]
        for _ in range(8):
            cy, cx = rng.integers(0, h), rng.integers(0, w)
            x += np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / 18.0).astype(np.float32)
    f = c[name]
    xd = torch.from_numpy(x).cuda()
    d, B, lap = detect.blur_laplacian_detect(xd, f, frac=0.5, return_fields=True)
    lap = lap.cpu().numpy()
    Bref, Lref, (ys, xs, vs, thr) = O.pipeline(x, f, frac=0.5)
    s = np.abs(Lref).max()
    e = np.abs(lap - Lref)
    i = np.unravel_index(e.argmax(), e.shape)
    ex, bad = compare_blobs(d.as_set(), set(zip(ys.tolist(), xs.tolist())), Lref, thr)
    ts = []
    for env in (None, "1"):
        if env:
            os.environ["VMF_NO_FIRTC"] = "1"
        else:
            os.environ.pop("VMF_NO_FIRTC", None)
        for _ in range(2):
            detect.blur_laplacian_detect(xd, f, frac=0.5)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            detect.blur_laplacian_detect(xd, f, frac=0.5)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) / 5 * 1e3)
    os.environ.pop("VMF_NO_FIRTC", None)
    print(f"{name:9s} {h}x{w}: L err {e.max() / s:.2e} at {i}, rows0/H-1 {e[0].max() / s:.1e}/"
          f"{e[-1].max() / s:.1e} cols0/W-1 {e[:, 0].max() / s:.1e}/{e[:, -1].max() / s:.1e}, "
          f"blobs gpu {d.count} ref {len(ys)} bad {len(bad)} exempt {ex} | ms tc {ts[0]:.3f} "
          f"fp64 {ts[1]:.3f}", flush=True)
