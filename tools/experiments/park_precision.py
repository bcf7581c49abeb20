"""How much precision do the design's rounding points cost?  numpy emulation
of the hot path with fp32 rounding inserted at: T (row-pass output), the
parked backward part of either pass, B (blur) before the Laplacian.
Error metric: max|L - L_ref| / max|L_ref| (parity tolerance 1e-4)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np
from oracle import oracle as O
from paper_1912_07133_b200 import filters, synth

f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)


def iir_lines(x, f, park32=False, out32=True):
    """rows of x (lines x n): DF-II fp64 like the reference, optional fp32
    parking of sign*y- and fp32 output."""
    b = np.array(f.b_plus); a = np.array(f.a_plus); k = len(a)
    M, n = x.shape
    asum = 1 + a.sum()
    sign = 1.0 if f.parity == "sym" else -1.0
    s = np.repeat(x[:, -1:] / asum, k, axis=1)
    ym = np.empty_like(x)
    for t in range(n - 1, -1, -1):
        ym[:, t] = s @ b
        wn = x[:, t] - s @ a
        s = np.concatenate([wn[:, None], s[:, :-1]], axis=1)
    p = sign * ym
    if park32:
        p = f32(p)
    s = np.repeat(x[:, :1] / asum, k, axis=1)
    out = np.empty_like(x)
    for t in range(n):
        out[:, t] = (f.b_zero * x[:, t] + s @ b) + p[:, t]
        wn = x[:, t] - s @ a
        s = np.concatenate([wn[:, None], s[:, :-1]], axis=1)
    return f32(out) if out32 else out


def run(x, f, label):
    x = f32(x)
    Lref = O.laplacian(O.blur(x, f))
    m = np.abs(Lref).max()
    variants = {
        "v1 (T32, B32)": dict(rp=False, cp=False, b32=True),
        "T32, B64": dict(rp=False, cp=False, b32=False),
        "row park32, B64": dict(rp=True, cp=False, b32=False),
        "row park32, B32": dict(rp=True, cp=False, b32=True),
        "row+col park32, B64": dict(rp=True, cp=True, b32=False),
    }
    for name, v in variants.items():
        T = iir_lines(x, f, park32=v["rp"], out32=True)
        B = iir_lines(T.T.copy(), f, park32=v["cp"], out32=v["b32"]).T
        L = O.laplacian(B)
        print(f"{label:24s} {name:22s} err/max|L| = {np.abs(L - Lref).max() / m:.2e}   max|L|={m:.3e}",
              flush=True)


if __name__ == "__main__":
    cat = filters.catalog()
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    x3 = synth.config3_frame(n)
    for s in ("rp2", "rp4", "rp32"):
        run(x3, cat[s], f"config3/{n}/{s}")
    x5 = synth.config5_frame(n)
    run(x5, cat["bw48"], f"config5/{n}/bw48")
    run(x5, cat["rp32"], f"config5/{n}/rp32")
