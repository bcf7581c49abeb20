"""Per-tile role timeline of the tensor-core FIR row / column pass, CTA 0
(build/abl/libtctl.so, built with -DVMF_TC_TL).  Stamps per tile: 0 first
slice issued, 1 last slice issued (producer), 2 MMA start, 3 MMA issue done,
4 epilogue start, 5 epilogue done."""
import ctypes as C
import os
import sys

import numpy as np

os.environ["VMF_LIB_PATH"] = os.path.abspath("build/abl/libtctl.so")
sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1912_07133_b200 import _lib, detect, filters, synth  # noqa: E402

c = filters.catalog()
x = torch.from_numpy(synth.config3_frame(4096)).cuda()
L = _lib.lib()
buf = np.zeros(1024, np.uint64)
for name in sys.argv[1:] or ["g2_k8", "g32_k128"]:
    f = c[name]
    for _ in range(3):
        detect.blur_laplacian_detect(x, f, frac=0.5)
    torch.cuda.synchronize()
    L.vmf_debug_tctl(buf.ctypes.data)  # (the column pass of the last call)
    t = buf.astype(np.int64).reshape(128, 8)[:, :6]
    n = int((t[:, 5] > 0).sum())
    t0 = t[0, 0]
    print(name, "tiles", n)
    for i in range(n):
        print("  tile %2d: issue %7.2f..%7.2f  mma %7.2f..%7.2f  epi %7.2f..%7.2f us" %
              tuple([i] + [(v - t0) / 1e3 for v in t[i, :6]]))
    sl = buf.astype(np.int64)[512:512 + 96 * 5].reshape(96, 5)
    print("  slice: tma issue -> full -> converted -> mma sees -> mma committed (us from tile 0)")
    for g in range(0, 40):
        if sl[g, 0] == 0:
            break
        print("   %2d: %s" % (g, "  ".join("%7.2f" % ((v - t0) / 1e3) for v in sl[g])))
