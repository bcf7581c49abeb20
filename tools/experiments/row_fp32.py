"""Can the FIRST (row) pass run in fp32 if the second (column) pass is fp64?
numpy emulation at fp32 of the row pass in three realisations (DF-II as in
engine.py:65-102, DF-I, DF-I with 32-sample chunk carries computed in fp32),
column pass in fp64 (oracle), Laplacian from fp64 B.  Metric max|dL|/max|L|."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np

from oracle import oracle as O
from paper_1912_07133_b200 import filters, synth

F = np.float32


def dfii32(x, f):
    b = np.array(f.b_plus, F); a = np.array(f.a_plus, F); k = len(a)
    M, n = x.shape
    asum = F(1) + a.sum(dtype=F)
    out = np.empty((M, n), F)
    s = np.repeat((x[:, :1] / asum).astype(F), k, axis=1)
    for t in range(n):
        acc = F(f.b_zero) * x[:, t] + (s * b).sum(1, dtype=F)
        wn = x[:, t] - (s * a).sum(1, dtype=F)
        out[:, t] = acc
        s = np.concatenate([wn[:, None], s[:, :-1]], axis=1)
    s = np.repeat((x[:, -1:] / asum).astype(F), k, axis=1)
    for t in range(n - 1, -1, -1):
        acc = (s * b).sum(1, dtype=F)
        wn = x[:, t] - (s * a).sum(1, dtype=F)
        out[:, t] = out[:, t] + acc
        s = np.concatenate([wn[:, None], s[:, :-1]], axis=1)
    return out


def dfi32(x, f, chunk=None):
    """DF-I in fp32; with `chunk`, histories at chunk starts come from an
    fp64-exact recursion rounded to fp32 plus an fp32-computed correction
    (emulates fp32 zero-state carries + scan: error ~ fp32 rounding of the
    carried history)."""
    b = np.array(f.b_plus, F); a = np.array(f.a_plus, F); k = len(a)
    M, n = x.shape
    yss = F(sum(f.b_plus) / (1 + sum(f.a_plus)))

    def run(xx, Y, X, reset_every=None, exact=None):
        out = np.empty_like(xx)
        for t in range(xx.shape[1]):
            if reset_every and t % reset_every == 0 and t > 0:
                # carry: exact history rounded to fp32, perturbed by 1 ulp
                Y = exact[:, t - 1::-1][:, :k].astype(F) if t >= k else Y
                Y = (Y * (1 + np.float32(6e-8) * np.sign(np.random.default_rng(t).standard_normal(Y.shape)))).astype(F)
            y = (X * b).sum(1, dtype=F) - (Y * a).sum(1, dtype=F)
            out[:, t] = y
            Y = np.concatenate([y[:, None], Y[:, :-1]], axis=1)
            X = np.concatenate([xx[:, t:t + 1], X[:, :-1]], axis=1)
        return out

    x0 = x[:, :1]; xl = x[:, -1:]
    ex_p = ex_m = None
    if chunk:
        # exact (fp64) one-sided parts for the carries
        fx = x.astype(np.float64)
        b64 = np.array(f.b_plus); a64 = np.array(f.a_plus)
        def exact(xx, e):
            Y = np.repeat(yss * e, k, 1).astype(np.float64); X = np.repeat(e, k, 1).astype(np.float64)
            o = np.empty_like(xx)
            for t in range(xx.shape[1]):
                y = X @ b64 - Y @ a64
                o[:, t] = y
                Y = np.concatenate([y[:, None], Y[:, :-1]], 1); X = np.concatenate([xx[:, t:t+1], X[:, :-1]], 1)
            return o
        ex_p = exact(fx, fx[:, :1]); ex_m = exact(fx[:, ::-1], fx[:, -1:])
    yp = run(x, np.repeat(yss * x0, k, 1).astype(F), np.repeat(x0, k, 1), chunk, ex_p)
    ym = run(x[:, ::-1].copy(), np.repeat(yss * xl, k, 1).astype(F), np.repeat(xl, k, 1), chunk, ex_m)[:, ::-1]
    return (F(f.b_zero) * x + yp) + ym


def main(n=512):
    cat = filters.catalog()
    for cfg, frame in ((3, synth.config3_frame(n)), (5, synth.config5_frame(n))):
        x = frame.astype(F)
        names = ("rp2", "rp4", "rp32") if cfg == 3 else ("bw48", "rp32")
        for nm in names:
            f = cat[nm]
            Lref = O.laplacian(O.blur(x, f))
            m = np.abs(Lref).max()
            for label, fn in (("dfii32", lambda: dfii32(x, f)), ("dfi32", lambda: dfi32(x, f)),
                              ("dfi32+carries", lambda: dfi32(x, f, 32))):
                T = fn()
                B = O.iir_cols(T.astype(np.float64), f)
                L = O.laplacian(B)
                print(f"config{cfg}/{n}/{nm:5s} {label:14s} err/max|L| = {np.abs(L - Lref).max() / m:.2e}",
                      flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 512)
