"""Golden IIR designs from the reference's own design code (design.py),
used by tests/test_design.py to pin paper_1912_07133_b200.design.

Run HERE, where /root/reference exists:   python tests/golden/make_design_golden.py
The reference package is imported from a scratch copy (nothing is written
into /root/reference).  Output: tests/golden/design_golden.json, one entry
per design call: b_plus, a_plus, b_zero, parity (or the exception the
reference raised); for the FIR designs the taps, parity and d of each kernel.
"""
import json
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SCRATCH = "/tmp/vmf_refpkg"

CALLS = (
    [f"repeated_pole_blur({s})" for s in (1.0, 1.25, 2.5, 5.0, 7.0, 10.0, 20.0, 40.0, 64.0)]
    + [f"repeated_pole_blur(6.0, {ld}, {lp})" for ld, lp in
       ((1, 0), (2, 0), (1, 1), (2, 1), (2, 2), (3, 1), (1, 4), (3, 3), (4, 2))]
    + [f"butterworth_blur({s})" for s in (1.0, 2.0, 3.0, 8.0, 16.0, 32.0, 64.0)]
    + [f"butterworth_blur(8.0, {ld})" for ld in (2, 3)]
    + [f"butterworth_appendix({lam})" for lam in (1.0, 2.0, 4.0, 10.0, 30.0)]
    + [f"blunt_exponential_blur({lam}, {k})" for lam in (1.0, 3.0, 12.0) for k in (1, 2, 3, 4)]
)
FIR_CALLS = (
    [f"interp_diff({d})" for d in range(9)]
    + [f"fir_vm_bank({D}, {lp}, '{mode}')" for D in (3, 5, 7, 9)
       for mode, lp in (("behind_blur", 2), ("standalone", 1), ("standalone", 2))]
    + [f"colored_sg_blur({s}, {ld})" for s, ld in ((1.0, 1), (2.0, 1), (4.5, 1), (2.0, 2), (3.5, 2))]
)


def main():
    if not os.path.isdir(SCRATCH):
        shutil.copytree("/root/reference/pkg", SCRATCH)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/vmf_numba_cache")
    sys.path.insert(0, os.path.join(SCRATCH, "src"))
    from vmfilt import design  # noqa: F401

    out = {}
    for call in CALLS:
        try:
            f = eval("design." + call)
        except Exception as exc:  # the reference's own rejection is golden too
            out[call] = {"error": type(exc).__name__, "message": str(exc)}
            continue
        out[call] = {"b_plus": list(f.b_plus), "a_plus": list(f.a_plus), "b_zero": f.b_zero,
                     "parity": f.parity}
    for call in FIR_CALLS:
        f = eval("design." + call)
        ks = f if isinstance(f, list) else [f]
        out[call] = {"fir": [{"taps": list(k.taps), "parity": k.parity, "d": k.d} for k in ks]}
    with open(os.path.join(HERE, "design_golden.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(len(out), "designs")


if __name__ == "__main__":
    main()
