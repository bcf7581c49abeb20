"""Generate the golden vectors that pin the oracle (tests/test_oracle.py).

Run HERE, where /root/reference exists:   python tests/golden/make_golden.py
It imports the reference package `vmfilt` from a scratch copy (NUMBA_CACHE_DIR
redirected, nothing written into /root/reference) and records the outputs of
its own hot-path functions on small seeded inputs:

  engine.iir_rows / iir_cols      engine.py:137-158
  engine.conv_rows / conv_cols    engine.py:112-126
  engine.apply_cols(apply_rows()) engine.py:161-174
  engine.derivative_field         engine.py:205-228  (order 3: D10 D01 D20 D02 D11)

Filters come from the reference's design code via paper_1912_07133_b200/data/
catalog.json (itself produced by tools/make_catalog.py).  Output:
tests/golden/golden.npz (float64; a few hundred KB).
"""
import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
SCRATCH = "/tmp/vmf_refpkg"


def main():
    if not os.path.isdir(SCRATCH):
        shutil.copytree("/root/reference/pkg", SCRATCH)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/vmf_numba_cache")
    sys.path.insert(0, os.path.join(SCRATCH, "src"))
    sys.path.insert(0, REPO)
    from vmfilt import engine, design
    from vmfilt.polyz import ThreePartIIR
    from paper_1912_07133_b200 import filters as F

    cat = F._catalog_raw()

    def ref_stage(name):
        e = cat[name]
        if e["type"] == "iir":
            return ThreePartIIR(tuple(e["b_plus"]), tuple(e["a_plus"]), e["b_zero"], e["parity"])
        return design.FirKernel(tuple(e["taps"]), e["parity"], e["d"])

    rng = np.random.default_rng(20191217)
    inputs = {
        "rand": rng.standard_normal((40, 56)),
        "tall": rng.random((97, 13)),
        "step": np.vstack([np.r_[[2.0] * 25, [5.0] * 25]] * 3),
        "const": np.full((20, 31), 3.7),
        "minrow": rng.random((3, 7)),       # w = 2K+1 for K = 3 (engine.py:139)
        "mincol": rng.random((7, 5)),
        "f32": rng.random((33, 45)).astype(np.float32).astype(np.float64),
        "u16": np.round(rng.uniform(0, 4095, (24, 40))),
    }
    out = {f"in/{k}": v for k, v in inputs.items()}
    iirs = ["rp4", "rp4_k2", "rp32", "rp1.5", "bw6", "bw48", "bwapp6", "blunt4", "rp4_k4"]
    firs = ["g1.5_k8", "g4_k16", "sg3.2", "vm_bank3_1", "vm_bank3_2"]
    for iname in ("rand", "tall", "step", "const", "minrow", "mincol", "f32", "u16"):
        x = inputs[iname]
        h, w = x.shape
        for fname in iirs:
            f = ref_stage(fname)
            if w >= 2 * f.k + 1:
                out[f"iir_rows/{fname}/{iname}"] = engine.iir_rows(x, f)
            if h >= 2 * f.k + 1:
                out[f"iir_cols/{fname}/{iname}"] = engine.iir_cols(x, f)
            if min(h, w) >= 2 * f.k + 1:
                out[f"blur/{fname}/{iname}"] = engine.apply_cols(engine.apply_rows(x, f), f)
        for fname in firs:
            k = ref_stage(fname)
            if len(k.taps) <= w:
                out[f"conv_rows/{fname}/{iname}"] = engine.conv_rows(x, k)
            if len(k.taps) <= h:
                out[f"conv_cols/{fname}/{iname}"] = engine.conv_cols(x, k)
            if len(k.taps) <= min(h, w) and fname.startswith(("g", "sg")):
                out[f"blur/{fname}/{iname}"] = engine.apply_cols(engine.apply_rows(x, k), k)
    for fname in ("rp4", "g1.5_k8", "bw6"):
        for iname in ("rand", "f32"):
            fld = engine.derivative_field(inputs[iname], ref_stage(fname), 3)
            for key in ((1, 0), (0, 1), (2, 0), (0, 2), (1, 1)):
                out[f"field/{fname}/{iname}/{key[0]}{key[1]}"] = fld[key]
    # gaussian_fir restatement pin (design.py:297-334)
    for s, d, k in ((1.5, 0, 8), (4.0, 0, 16), (2.0, 1, 10), (3.0, 2, 12)):
        out[f"gauss/{s}/{d}/{k}"] = np.asarray(design.gaussian_fir(s, d, k).taps)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
