"""Seed sweep of tests/test_gpu_parity.py::test_fused_path_odd_shapes inputs
(debug helper): prints every blob-set difference that is not a near-tie."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_1912_07133_b200 import detect, filters  # noqa: E402
from oracle import oracle as O  # noqa: E402
from parity import compare_blobs, TOL_REL  # noqa: E402

cat = filters.catalog()
shape = tuple(int(v) for v in sys.argv[1].split("x")) if len(sys.argv) > 1 else (1000, 33)
names = sys.argv[2].split(",") if len(sys.argv) > 2 else ["rp4"]
nseed = int(sys.argv[3]) if len(sys.argv) > 3 else 200
h, w = shape
nbad = 0
start = int(sys.argv[4]) if len(sys.argv) > 4 else 0
for name in names:
    for seed in range(start, start + nseed):
        rng = np.random.default_rng(seed)
        x = (0.05 * rng.standard_normal((h, w))).astype(np.float32)
        for _ in range(6):
            cy, cx = rng.integers(0, h), rng.integers(0, w)
            yy, xx = np.ogrid[:h, :w]
            x += np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / 18.0).astype(np.float32)
        dets, blur, lap = detect.blur_laplacian_detect(torch.as_tensor(x).cuda(), cat[name],
                                                       frac=0.5, return_fields=True)
        B, L, (ys, xs, vs, thr) = O.pipeline(x, cat[name], frac=0.5, lap_scale=1.0)
        got, want = dets.as_set(), set(zip(ys.tolist(), xs.tolist()))
        ex, bad = compare_blobs(got, want, L, thr)
        if bad:
            nbad += 1
            lg = lap.cpu().numpy()
            for (y, xq) in bad:
                print(name, seed, (y, xq), "gpu" if (y, xq) in got else "ref",
                      "L_ref", L[y, xq], "L_gpu", lg[y, xq], "thr", thr, "tol", TOL_REL * np.abs(L).max(),
                      "ref nb", np.round(L[max(y-1,0):y+2, max(xq-1,0):xq+2], 6).tolist(),
                      "gpu nb", np.round(lg[max(y-1,0):y+2, max(xq-1,0):xq+2], 6).tolist(),
                      "overflow", dets.overflow, "count", dets.count, len(want))
print("bad seeds", nbad)
