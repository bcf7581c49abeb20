"""fp32 column pass (vmf_colpass32.cu) against the oracle: L error per
filter / shape, blob sets, and timing of one fused scale."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O
from paper_1912_07133_b200 import detect, filters, synth
from tests.parity import compare_blobs

O.set_threads(O.max_threads())
c = filters.catalog()
cases = [("rp4", (512, 512)), ("rp4_k2", (512, 512)), ("rp4_k4", (300, 517)), ("bw6", (257, 389)),
         ("rp32", (4096, 4096)), ("rp2", (4096, 4096)), ("rp16", (4096, 4096)),
         ("bw48", (4096, 4096)), ("rp6", (2048, 2048)), ("rp8", (1000, 1033)), ("rp4", (67, 131)),
         ("rp4", (129, 64)), ("rp4", (1000, 33))]
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
    d, lap = None, None
    d, B, lap = detect.blur_laplacian_detect(x, f, frac=0.5, return_fields=True)
    Bref, Lref, (ys, xs, vs, thr) = O.pipeline(x, f, frac=0.5)
    s = np.abs(Lref).max()
    e = np.abs(lap - Lref)
    i = np.unravel_index(e.argmax(), e.shape)
    ex, bad = compare_blobs(d.as_set(), set(zip(ys.tolist(), xs.tolist())), Lref, thr)
    print(f"{name:7s} {h}x{w}: L err {e.max() / s:.2e} at {i}, rows0/H-1 {e[0].max() / s:.1e}/"
          f"{e[-1].max() / s:.1e}, blobs gpu {d.count} ref {len(ys)} bad {len(bad)} exempt {ex}",
          flush=True)
