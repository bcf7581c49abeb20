"""Numpy prototype of the fp32 "Laplacian-first" column pass, chunked the
way the CUDA kernels are (vmf_colpass32.cu): every step in float32.

  U = 5-point Laplacian of the row-pass output T (replicate edges, clamped
      rows past the bottom, so padded rows carry U = D20 T(H-1)),
  state-space modal realisation of the causal part  y+(n) = c . u(n-1),
      u(n) = A u(n-1) + b U(n)   (Jordan chain for a repeated real pole,
      rotation for a complex pair), the anticausal part mirrored,
  bands of 64 rows: zero-state band carries by folded sample pairs, a scan
      over bands with A^64, steady-state starts from D20 T of rows 0 / H-1,
  per band a backward walk (parked) and a forward walk producing L directly,
      plus L at rows r0-1 and r1 via c A^-1 (the NMS halo rows),
  boundary corrections at rows 0 and H-1 from band partial sums of
      h(m) G(m), G(m) = T(m) - T(m-1).
Compared with the oracle's fp64 pipeline (blur -> Laplacian)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np

from oracle import oracle as O
from paper_1912_07133_b200 import filters, synth

F = np.float32
BAND = 64


def modal(f):
    """-> (A, b, c) float64 with y+(n) = c.u(n-1), u(n) = A u(n-1) + b x(n)."""
    bp, ap = np.array(f.b_plus), np.array(f.a_plus)
    k = len(ap)
    p = -ap[0] / k
    if np.allclose(np.poly([p] * k)[1:], ap, rtol=0, atol=1e-13):
        A = p * np.tril(np.ones((k, k)))
        b = np.ones(k)
    elif k == 2:
        r = np.roots(np.r_[1.0, ap])
        pc = r[0] if r[0].imag > 0 else r[1]
        A = np.array([[pc.real, -pc.imag], [pc.imag, pc.real]])
        b = np.array([1.0, 0.0])
    else:
        raise ValueError("no modal realisation")
    # c from the impulse response: h(m) = c A^(m-1) b, m = 1..k (k equations)
    h = np.zeros(k + 1)
    s = np.zeros(k)
    for t in range(k + 1):  # DF-II impulse response of the reference
        x = 1.0 if t == 0 else 0.0
        h[t] = bp @ s
        s = np.r_[x - ap @ s, s[:-1]]
    M = np.array([np.linalg.matrix_power(A, m - 1) @ b for m in range(1, k + 1)])
    c = np.linalg.solve(M, h[1:k + 1])
    return A, b, c


def lap5(T):
    Tu = np.vstack([T[:1], T[:-1]])
    Td = np.vstack([T[1:], T[-1:]])
    Tl = np.hstack([T[:, :1], T[:, :-1]])
    Tr = np.hstack([T[:, 1:], T[:, -1:]])
    return ((Tl - T) + (Tr - T)) + ((Tu - T) + (Td - T))


def colpass32(T32, f, lsc=1.0):
    A64, b64, c64 = modal(f)
    k = len(b64)
    sign = 1.0 if f.parity == "sym" else -1.0
    H, W = T32.shape
    NB = -(-H // BAND)
    Hp = NB * BAND
    T = T32.astype(F)
    Tp = np.vstack([T, np.repeat(T[-1:], Hp - H, axis=0)])  # clamped rows
    U = lap5(np.vstack([Tp, Tp[-1:]]))[:Hp].astype(F)  # replicate at the padded end too
    # (rows >= H of U = D20 T(H-1): the vertical part vanishes on clamped rows)
    A, b, c = A64.astype(F), b64.astype(F), c64.astype(F)
    Wk = np.array([np.linalg.matrix_power(A64, t) @ b64 for t in range(BAND)])  # A^t b
    # ---- band carries (folded pairs) -------------------------------------
    half = BAND // 2
    wp = (0.5 * (Wk[:half] + Wk[::-1][:half])).astype(F)   # (W(t) + W(L-1-t))/2
    wq = (0.5 * (Wk[::-1][:half] - Wk[:half])).astype(F)   # (W(L-1-t) - W(t))/2
    zf = np.zeros((NB, k, W), F)
    zb = np.zeros((NB, k, W), F)
    for bnd in range(NB):
        blk = U[bnd * BAND:(bnd + 1) * BAND]
        P = np.zeros((k, W), F)
        Q = np.zeros((k, W), F)
        for t in range(half):
            S = blk[t] + blk[BAND - 1 - t]
            D = blk[t] - blk[BAND - 1 - t]
            P = P + wp[t][:, None] * S
            Q = Q + wq[t][:, None] * D
        zf[bnd] = P + Q
        zb[bnd] = P - Q
    # ---- scan over bands ---------------------------------------------------
    AL = np.linalg.matrix_power(A64, BAND).astype(F)
    Iss = np.linalg.solve(np.eye(k) - A64, b64).astype(F)  # u_ss = Iss * e
    Tl = np.hstack([T[:, :1], T[:, :-1]])
    Tr = np.hstack([T[:, 1:], T[:, -1:]])
    D20 = (Tl - T) + (Tr - T)
    e_top, e_bot = D20[0], D20[-1]
    uf_start = np.zeros((NB, k, W), F)  # uf(r0 - 1)
    ub_start = np.zeros((NB, k, W), F)  # ub(r1)
    s = Iss[:, None] * e_top[None, :]
    for bnd in range(NB):
        uf_start[bnd] = s
        s = AL @ s + zf[bnd]
    s = Iss[:, None] * e_bot[None, :]
    for bnd in range(NB - 1, -1, -1):
        ub_start[bnd] = s
        s = AL @ s + zb[bnd]
    # ---- boundary corrections ---------------------------------------------
    hm = np.array([c64 @ np.linalg.matrix_power(A64, m - 1) @ b64 for m in range(1, Hp + 1)])
    hm = np.r_[0.0, hm].astype(F)  # hm[m] = h(m)
    G = np.vstack([np.zeros((1, W), F), Tp[1:] - Tp[:-1]])  # G(r) = T(r) - T(r-1)
    ctop = np.zeros(W, F)
    cbot = np.zeros(W, F)
    for bnd in range(NB):  # band partials, summed in band order
        pt = np.zeros(W, F)
        pb = np.zeros(W, F)
        for r in range(bnd * BAND, (bnd + 1) * BAND):
            if 1 <= r < H:
                pt = pt + hm[r] * G[r]
                pb = pb + hm[H - r] * G[r]
        ctop = ctop + pt
        cbot = cbot + pb
    # ---- per band walks ----------------------------------------------------
    cinv = (c64 @ np.linalg.inv(A64)).astype(F)
    e1 = F(cinv.astype(np.float64) @ b64)
    Lx = np.zeros((Hp, W), F)
    halo_top = np.zeros((NB, W), F)  # L(r0 - 1)
    halo_bot = np.zeros((NB, W), F)  # L(r1)
    b0, sg, ls = F(f.b_zero), F(sign), F(lsc)
    Uext = np.vstack([U, U[-1:]])
    for bnd in range(NB):
        r0, r1 = bnd * BAND, (bnd + 1) * BAND
        park = np.zeros((BAND, W), F)
        s = ub_start[bnd].copy()
        for r in range(r1 - 1, r0 - 1, -1):
            park[r - r0] = c @ s
            s = A @ s + b[:, None] * U[r]
        ym_above = c @ s                      # y-(r0 - 1)
        s = uf_start[bnd].copy()
        if r0 > 0:
            yp_above = cinv @ s - e1 * U[r0 - 1]   # y+(r0 - 1)
            halo_top[bnd] = ls * (b0 * U[r0 - 1] + yp_above + sg * ym_above)
        for r in range(r0, r1):
            Lx[r] = ls * (b0 * U[r] + c @ s + sg * park[r - r0])
            s = A @ s + b[:, None] * U[r]
        if r1 < Hp:
            ym_below = cinv @ ub_start[bnd] - e1 * Uext[r1]   # y-(r1)
            halo_bot[bnd] = ls * (b0 * Uext[r1] + c @ s + sg * ym_below)
    L = Lx[:H].copy()
    L[0] = L[0] + ls * sg * ctop
    L[H - 1] = L[H - 1] - ls * cbot
    # halo rows must equal the neighbouring band's own rows
    hd = 0.0
    for bnd in range(1, NB):
        r0 = bnd * BAND
        if r0 - 1 < H:
            ref_row = L[r0 - 1]
            hd = max(hd, float(np.abs(halo_top[bnd] - ref_row).max()))
        if r0 < H:
            hd = max(hd, float(np.abs(halo_bot[bnd - 1] - L[r0]).max()))
    return L, hd


def run(name, x):
    f = filters.catalog()[name]
    T32 = O.iir_rows(x, f).astype(np.float32)
    Lref = O.laplacian(O.blur(x, f))
    s = np.abs(Lref).max()
    L, hd = colpass32(T32, f)
    e = np.abs(L.astype(np.float64) - Lref).max() / s
    cur = np.abs(O.laplacian(O.iir_cols(T32.astype(np.float64), f)) - Lref).max() / s
    print(f"{name:8s} fp32 chunked {e:.2e}  (fp64 column pass on the same T: {cur:.2e})  "
          f"halo-row mismatch {hd / s:.1e}", flush=True)
    return e


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    x3 = synth.config3_frame(n)
    for nm in ("rp2", "rp4", "rp8", "rp16", "rp32", "rp4_k2", "rp4_k4"):
        run(nm, x3)
    run("bw48", synth.config5_frame(n))
    run("bw6", x3)
    run("rp6", synth.config4_stream(1, n)[0].astype(np.float32))
    run("rp4", x3[: n - 37, : n - 5])  # ragged: a short last band
