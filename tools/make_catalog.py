"""Design every filter the five BASELINE configs (and the parity tests) use,
with the reference's own design code, and write the coefficients as JSON.

Run HERE (container with /root/reference); the output travels with the repo,
so the GPU box never needs the reference or mpmath.  The reference is imported
from a scratch copy with NUMBA_CACHE_DIR redirected so nothing is written into
/root/reference.

    python tools/make_catalog.py  ->  paper_1912_07133_b200/data/catalog.json

Design entry points (file:line under /root/reference/pkg/src/vmfilt/):
repeated_pole_blur design.py:480, butterworth_blur design.py:511,
gaussian_fir design.py:297, colored_sg_blur design.py:337,
fir_vm_bank design.py:250, blunt_exponential_blur design.py:520,
butterworth_appendix design.py:559.
"""
import json
import os
import shutil
import sys
import time

REF = "/root/reference/pkg"
SCRATCH = "/tmp/vmf_refpkg"


def import_reference():
    if not os.path.isdir(SCRATCH):
        shutil.copytree(REF, SCRATCH)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/vmf_numba_cache")
    sys.path.insert(0, os.path.join(SCRATCH, "src"))
    import vmfilt  # noqa: F401
    return vmfilt


def main(out=None):
    vm = import_reference()
    from vmfilt import design
    out = out or os.path.join(os.path.dirname(__file__), "..",
                              "paper_1912_07133_b200", "data", "catalog.json")
    cat = {}

    def iir(name, f, how):
        cat[name] = {"type": "iir", "b_plus": list(f.b_plus), "a_plus": list(f.a_plus),
                     "b_zero": f.b_zero, "parity": f.parity, "design": how}

    def fir(name, f, how):
        cat[name] = {"type": "fir", "taps": list(f.taps), "parity": f.parity,
                     "d": f.d, "design": how}

    t0 = time.time()
    for s in (1.5, 2.0, 3.0, 4.0, 6.0, 8.0, 12.0, 16.0, 24.0, 32.0):
        iir(f"rp{s:g}", design.repeated_pole_blur(s), f"repeated_pole_blur({s})")
    iir("rp4_k2", design.repeated_pole_blur(4.0, 1, 1), "repeated_pole_blur(4.0, 1, 1)")
    iir("rp4_k4", design.repeated_pole_blur(4.0, 1, 3), "repeated_pole_blur(4.0, 1, 3)")
    for s in (4.0, 6.0, 48.0):
        iir(f"bw{s:g}", design.butterworth_blur(s), f"butterworth_blur({s})")
    iir("bwapp6", design.butterworth_appendix(6.0), "butterworth_appendix(6.0)")
    iir("blunt4", design.blunt_exponential_blur(4.0), "blunt_exponential_blur(4.0)")
    for s in (2.0, 4.0, 8.0, 16.0, 32.0):
        k = int(4 * s)
        fir(f"g{s:g}_k{k}", design.gaussian_fir(s, 0, k), f"gaussian_fir({s}, 0, {k})")
    fir("g1.5_k8", design.gaussian_fir(1.5, 0, 8), "gaussian_fir(1.5, 0, 8)")
    for s in (3.0, 6.0, 12.0, 24.0):
        k = int(round(5 * s))
        fir(f"g{s:g}_k{k}", design.gaussian_fir(s, 0, k), f"gaussian_fir({s}, 0, {k})")
    fir("sg3.2", design.colored_sg_blur(3.2), "colored_sg_blur(3.2)")
    bank = design.fir_vm_bank(3, cascade_mode="behind_blur")
    for i, b in enumerate(bank):
        fir(f"vm_bank3_{i}", b, f"fir_vm_bank(3)[{i}]")
    print(f"fast designs {time.time() - t0:.1f}s", flush=True)
    t0 = time.time()
    fir("sg38.4", design.colored_sg_blur(38.4), "colored_sg_blur(38.4)")
    print(f"sg38.4 {time.time() - t0:.1f}s", flush=True)
    with open(out, "w") as fh:
        json.dump(cat, fh, indent=1)
        fh.write("\n")
    print("wrote", out, len(cat), "filters")


if __name__ == "__main__":
    main(*sys.argv[1:])
