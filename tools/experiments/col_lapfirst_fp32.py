"""Column pass in fp32 on the Laplacian of T ("Laplacian first").

The reference computes B = C(T) (column IIR, steady-state starts), then
L = D20(B) + D02(B) with replicate edges.  By linearity and shift invariance
on the replicate-extended column:

    L = C0(U) + corrections at rows 0 and H-1,
    U = 5-point Laplacian of T with replicate edges (zero outside the rows),
    C0 = the same three-part column filter with ZERO initial states,
    L(0)   += sign * sum_{m>=1} h+(m) G(m)          (G(m) = T(m) - T(m-1))
    L(H-1) -=        sum_{m>=1} h+(m) G(H-m)

U and G are small (differences), so an fp32 recursion over U has errors
relative to |L|, not to |B|.  This script measures that claim: the row pass
output T (fp64 recursion, rounded to fp32 -- what the GPU stores) goes through
fp32 realisations of the column filter, and L is compared with the oracle's
fp64 pipeline.  Realisations:
  dfi     -- DF-I recursion in fp32 (the reference structure)
  modal   -- repeated real pole p: cascade u1 = p u1 + x, u2 = p u2 + u1, ...
             (Jordan form), y+ = d . u(n-1); complex pair: coupled rotation
             (modal form); coefficients rounded to fp32.
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np

from oracle import oracle as O
from paper_1912_07133_b200 import filters, synth

F = np.float32


def impulse(f, n):
    b, a = np.array(f.b_plus), np.array(f.a_plus)
    k = len(a)
    h = np.zeros(n)
    s = np.zeros(k)  # DF-II state w(n-1..n-k)
    for t in range(n):
        x = 1.0 if t == 0 else 0.0
        y = b @ s
        w = x - a @ s
        s = np.r_[w, s[:-1]]
        h[t] = y
    return h  # h[0] = 0 (strictly causal)


def lap5_rep32(T):
    """5-point Laplacian of fp32 T with replicate edges, as differences."""
    T = T.astype(F)
    Tu = np.vstack([T[:1], T[:-1]])
    Td = np.vstack([T[1:], T[-1:]])
    Tl = np.hstack([T[:, :1], T[:, :-1]])
    Tr = np.hstack([T[:, 1:], T[:, -1:]])
    return ((Tl - T) + (Tr - T)) + ((Tu - T) + (Td - T))


def poles_of(f):
    a = np.array(f.a_plus)
    k = len(a)
    p = -a[0] / k
    rep = np.allclose(np.poly([p] * k)[1:], a, rtol=0, atol=1e-13)
    if rep:
        return "rep", p
    r = np.roots(np.r_[1.0, a])
    return "distinct", r


def modal_coeffs(f):
    """Partial fractions of the causal part N(w)/A(w) (w = z^-1, the DF-II
    output y+(n) = (b1 w + b2 w^2 + ...)/A(w) x = w N(w)/A(w) x)."""
    b = np.array(f.b_plus)
    kind, P = poles_of(f)
    k = len(b)
    if kind == "rep":
        p = P
        # N(w) = sum_j d_j (1 - p w)^{k-j}, j = 1..k  (d_j multiplies 1/(1-pw)^j)
        # solve by sampling w at k points
        ws = np.linspace(-0.5, 0.5, k)
        M = np.array([[(1 - p * w) ** (k - j) for j in range(1, k + 1)] for w in ws])
        N = np.array([np.polyval(b[::-1], w) for w in ws])
        d = np.linalg.solve(M, N)
        return kind, p, d
    # distinct: d_i = N(1/p_i) / prod_{j != i} (1 - p_j / p_i)
    d = []
    for i, pi in enumerate(P):
        w = 1 / pi
        num = np.polyval(b[::-1], w)
        den = np.prod([1 - pj * w for j, pj in enumerate(P) if j != i])
        d.append(num / den)
    return kind, P, np.array(d)


def causal32(U, f, real, reverse=False, e=None):
    """y+(n) = sum_{m>=1} h+(m) U(n-m) along axis 0, fp32, the history before
    row 0 being the constant row e (steady state)."""
    if reverse:
        return causal32(U[::-1], f, real, e=e)[::-1]
    H = U.shape[0]
    y = np.zeros_like(U, dtype=F)
    e = np.zeros(U.shape[1]) if e is None else np.asarray(e, np.float64)
    if real == "dfi":
        b = np.array(f.b_plus).astype(F)
        a = np.array(f.a_plus).astype(F)
        k = len(a)
        yss = np.sum(f.b_plus) / (1 + np.sum(f.a_plus))
        X = [e.astype(F) for _ in range(k)]
        Y = [(yss * e).astype(F) for _ in range(k)]
        for n in range(H):
            acc = np.zeros(U.shape[1], F)
            for m in range(k):
                acc = acc + b[m] * X[m]
            for m in range(k):
                acc = acc - a[m] * Y[m]
            y[n] = acc
            X = [U[n].astype(F)] + X[:-1]
            Y = [acc] + Y[:-1]
        return y
    kind, P, d = modal_coeffs(f)
    if kind == "rep":
        k = len(d)
        p = F(P)
        dF = d.astype(F)
        u = [(e / (1 - P) ** (j + 1)).astype(F) for j in range(k)]
        for n in range(H):
            acc = np.zeros(U.shape[1], F)
            for j in range(k):
                acc = acc + dF[j] * u[j]
            y[n] = acc
            prev = U[n].astype(F)
            for j in range(k):
                u[j] = p * u[j] + prev
                prev = u[j]
        return y
    # distinct poles: real ones first order, complex pairs coupled
    secs = []
    used = set()
    for i, pi in enumerate(P):
        if i in used:
            continue
        if abs(pi.imag) < 1e-14:
            secs.append(("r", F(pi.real), F(d[i].real)))
            used.add(i)
        else:
            j = next(j for j in range(len(P)) if j != i and j not in used and abs(P[j] - np.conj(pi)) < 1e-12)
            used |= {i, j}
            if pi.imag < 0:
                pi, di = P[j], d[j]
            else:
                di = d[i]
            secs.append(("c", F(pi.real), F(pi.imag), F(2 * di.real), F(-2 * di.imag)))
    st = []
    for s_ in secs:
        if s_[0] == "r":
            st.append([(e / (1 - float(s_[1]))).astype(F), None])
        else:
            v = e / (1 - (float(s_[1]) + 1j * float(s_[2])))
            st.append([v.real.astype(F), v.imag.astype(F)])
    for n in range(H):
        acc = np.zeros(U.shape[1], F)
        for s, S in zip(secs, st):
            if s[0] == "r":
                acc = acc + s[2] * S[0]
            else:
                acc = acc + s[3] * S[0] + s[4] * S[1]
        y[n] = acc
        x = U[n].astype(F)
        for s, S in zip(secs, st):
            if s[0] == "r":
                S[0] = s[1] * S[0] + x
            else:
                ur, ui = S
                S[0] = (s[1] * ur - s[2] * ui) + x
                S[1] = s[2] * ur + s[1] * ui
    return y


def lapfirst_L(T32, f, real):
    U = lap5_rep32(T32)
    sign = F(1.0 if f.parity == "sym" else -1.0)
    T = T32.astype(F)
    Tl = np.hstack([T[:, :1], T[:, :-1]])
    Tr = np.hstack([T[:, 1:], T[:, -1:]])
    D20 = (Tl - T) + (Tr - T)
    yp = causal32(U, f, real, e=D20[0])
    ym = causal32(U, f, real, reverse=True, e=D20[-1])
    L = F(f.b_zero) * U + yp + sign * ym
    # boundary corrections: dot products of G with h+ (fp32)
    H = T32.shape[0]
    h = impulse(f, min(H, 4096)).astype(F)
    T = T32.astype(F)
    G = np.vstack([np.zeros((1, T.shape[1]), F), T[1:] - T[:-1]])  # G(m) = T(m)-T(m-1), G(0)=0
    M = min(H - 1, len(h) - 1)
    top = np.zeros(T.shape[1], F)
    bot = np.zeros(T.shape[1], F)
    for m in range(1, M + 1):
        top = top + h[m] * G[m]
        bot = bot + h[m] * G[H - m]
    L[0] = L[0] + sign * top
    L[H - 1] = L[H - 1] - bot
    return L


def run(name, x, realisations=("dfi", "modal")):
    f = filters.catalog()[name]
    T32 = O.iir_rows(x, f).astype(np.float32)
    Lref = O.laplacian(O.blur(x, f))
    s = np.abs(Lref).max()
    # fp64 algebra check (exact arithmetic version of the same formula)
    out = {}
    for r in realisations:
        L = lapfirst_L(T32, f, r)
        e = np.abs(L.astype(np.float64) - Lref)
        out[r] = (e.max() / s, e[1:-1].max() / s)
    # current GPU-like reference: fp64 columns on the fp32 T
    Lcur = O.laplacian(O.iir_cols(T32.astype(np.float64), f))
    out["fp64-on-T32"] = (np.abs(Lcur - Lref).max() / s,)
    print(name, {k: tuple(f"{v:.2e}" for v in vs) for k, vs in out.items()}, flush=True)


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    x3 = synth.config3_frame(n)
    for nm in ("rp2", "rp4", "rp8", "rp16", "rp32", "rp4_k2", "rp4_k4"):
        run(nm, x3)
    run("bw48", synth.config5_frame(n))
    run("rp6", synth.config4_stream(1, n)[0].astype(np.float32))
