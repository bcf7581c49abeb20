"""Where does the fused path lose precision at 4096^2 / sigma 32?  Row pass
(T) vs column pass (B, L), error locations, against the oracle."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O
from paper_1912_07133_b200 import detect, engine, filters, synth

O.set_threads(O.max_threads())
c = filters.catalog()
x = synth.config3_frame(4096)
for name in sys.argv[1:] or ["rp32", "rp16"]:
    f = c[name]
    Tref = O.iir_rows(x, f)
    Bref = O.iir_cols(Tref, f)
    Lref = O.laplacian(Bref)
    sL, sB = np.abs(Lref).max(), np.abs(Bref).max()
    Tg = engine.iir_rows(x, f)
    eT = np.abs(Tg - Tref)
    print(name, "T err/max|T|", eT.max() / np.abs(Tref).max(), "at", np.unravel_index(eT.argmax(), eT.shape))
    L_fromTg = O.laplacian(O.iir_cols(Tg, f))
    print(name, "oracle cols on GPU T: L err", np.abs(L_fromTg - Lref).max() / sL)
    d, Bg, Lg = detect.blur_laplacian_detect(x, f, frac=0.5, return_fields=True)
    eB = np.abs(Bg - Bref)
    eL = np.abs(Lg - Lref)
    print(name, "fused B err/max|B|", eB.max() / sB, "at", np.unravel_index(eB.argmax(), eB.shape))
    i = np.unravel_index(eL.argmax(), eL.shape)
    print(name, "fused L err/max|L|", eL.max() / sL, "at", i, "Lref", Lref[i], "Lg", Lg[i])
    rows = eL.max(axis=1) / sL
    print(name, "L err by row: first 4", rows[:4], "last 4", rows[-4:], "interior max", rows[4:-4].max())
    print(name, "oracle Laplacian of GPU B: L err", np.abs(O.laplacian(Bg) - Lref).max() / sL)
    Tg2 = torch.from_numpy(Tg).cuda()
    Lc = engine.iir_cols(Tg2, f).cpu().numpy()
    print(name, "leaf iir_cols on GPU T vs oracle cols on GPU T", np.abs(Lc - O.iir_cols(Tg, f)).max() / sB)
