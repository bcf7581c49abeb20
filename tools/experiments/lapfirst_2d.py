"""Both passes "Laplacian first": the whole blur -> Laplacian path on the
5-point Laplacian of the input, in fp32 (numpy prototype of the design in
DESIGN.md §2).

Reference (replicate edges everywhere): T = R X (rows), B = C T (columns),
L = Lap5_rep(B).  On the 2-D replicate extension X_ext everything commutes:
    Lap5(B_full) = C R Lap5(X_ext),
so with U0 = Lap5(X_ext) (inside the image: Lap5_rep X; left / right of the
image: D02 X of column 0 / W-1, constant along the row; above / below: D20 X
of row 0 / H-1, zero beyond the columns):
    V   = R U0            row pass, steady starts eL(r) = D02 X(r, 0),
                          eR(r) = D02 X(r, W-1)
    Vt  = R0 D20 X(0, .)  (zero starts)  -- the rows above the image
    Vb  = R0 D20 X(H-1, .)               -- the rows below
    L   = C V             column pass, steady starts Vt(c) / Vb(c)
and the replicate rule differs from Lap5(B_full) only on the border:
    L(r, 0)   += kx_l(r) = C[dx_l](r),  dx_l(r) = s sum_m h(m) (X(r, m) - X(r, m-1))
    L(r, W-1) -= kx_r(r) = C[dx_r](r),  dx_r(r) =   sum_m h(m) (X(r, W-m) - X(r, W-1-m))
    L(0, c)   += ky_t(c) = R[dy_t](c),  dy_t(c) = s sum_m h(m) (X(m, c) - X(m-1, c))
    L(H-1, c) -= ky_b(c) = R[dy_b](c),  dy_b(c) =   sum_m h(m) (X(H-m, c) - X(H-1-m, c))
(C, R with steady-state starts; s = sign of the anticausal part).  kx is
folded into the column pass by adding dx_l(r) to V(r, 0) (and -dx_r to
V(r, W-1), the extensions likewise): C is linear.
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, os.path.dirname(__file__))
import numpy as np

from col_lapfirst_chunked import modal  # noqa: E402
from oracle import oracle as O
from paper_1912_07133_b200 import filters, synth

F = np.float32


def filt1d(x, f, dt, e_lo=None, e_hi=None, axis=1):
    """Three-part filter along `axis` in dtype dt (modal form), with the
    history before the line a constant e_lo (None: zero) and after it e_hi."""
    A, b, c = modal(f)
    A, b, c = A.astype(dt), b.astype(dt), c.astype(dt)
    k = len(b)
    sign = 1.0 if f.parity == "sym" else -1.0
    X = np.moveaxis(np.asarray(x, dt), axis, 0)
    n = X.shape[0]
    rest = X.shape[1:]
    Iss = np.linalg.solve(np.eye(k) - modal(f)[0], modal(f)[1]).astype(dt)
    lo = np.zeros(rest, dt) if e_lo is None else np.asarray(e_lo, dt)
    hi = np.zeros(rest, dt) if e_hi is None else np.asarray(e_hi, dt)
    u = (Iss.reshape((k,) + (1,) * len(rest)) * lo[None]).astype(dt)
    yp = np.empty_like(X)
    for t in range(n):
        yp[t] = np.tensordot(c, u, axes=1)
        u = (np.tensordot(A, u, axes=1) + b.reshape((k,) + (1,) * len(rest)) * X[t]).astype(dt)
    u = (Iss.reshape((k,) + (1,) * len(rest)) * hi[None]).astype(dt)
    ym = np.empty_like(X)
    for t in range(n - 1, -1, -1):
        ym[t] = np.tensordot(c, u, axes=1)
        u = (np.tensordot(A, u, axes=1) + b.reshape((k,) + (1,) * len(rest)) * X[t]).astype(dt)
    out = (dt(f.b_zero) * X + yp + dt(sign) * ym).astype(dt)
    return np.moveaxis(out, 0, axis)


def hvec(f, n):
    A, b, c = modal(f)
    return np.array([0.0] + [c @ np.linalg.matrix_power(A, m - 1) @ b for m in range(1, n)])


def lapfirst2d(x, f, dt=F):
    X = np.asarray(x, dt)
    H, W = X.shape
    s = dt(1.0 if f.parity == "sym" else -1.0)
    up = np.vstack([X[:1], X[:-1]]); dn = np.vstack([X[1:], X[-1:]])
    lf = np.hstack([X[:, :1], X[:, :-1]]); rt = np.hstack([X[:, 1:], X[:, -1:]])
    D20 = (lf - X) + (rt - X)
    D02 = (up - X) + (dn - X)
    U0 = D20 + D02
    h = hvec(f, max(H, W)).astype(dt)
    # row-direction border terms (per row), folded into V's edge columns
    Gx = np.hstack([np.zeros((H, 1), dt), X[:, 1:] - X[:, :-1]])  # Gx(r, m) = X(r,m) - X(r,m-1)
    dxl = s * (Gx[:, 1:] * h[1:W][None, :]).sum(axis=1, dtype=dt)
    dxr = (Gx[:, 1:][:, ::-1] * h[1:W][None, :]).sum(axis=1, dtype=dt)  # m -> X(W-m) - X(W-1-m)
    V = filt1d(U0, f, dt, e_lo=D02[:, 0], e_hi=D02[:, -1], axis=1)
    V[:, 0] += dxl
    V[:, -1] -= dxr
    Vt = filt1d(D20[:1], f, dt, axis=1)[0]
    Vb = filt1d(D20[-1:], f, dt, axis=1)[0]
    Vt[0] += dxl[0]; Vt[-1] -= dxr[0]
    Vb[0] += dxl[-1]; Vb[-1] -= dxr[-1]
    L = filt1d(V, f, dt, e_lo=Vt, e_hi=Vb, axis=0)
    # column-direction border terms (per column), after the column pass
    Gy = np.vstack([np.zeros((1, W), dt), X[1:] - X[:-1]])
    dyt = s * (Gy[1:] * h[1:H][:, None]).sum(axis=0, dtype=dt)
    dyb = (Gy[1:][::-1] * h[1:H][:, None]).sum(axis=0, dtype=dt)
    L[0] += filt1d(dyt[None], f, dt, e_lo=dyt[:1], e_hi=dyt[-1:], axis=1)[0]
    L[-1] -= filt1d(dyb[None], f, dt, e_lo=dyb[:1], e_hi=dyb[-1:], axis=1)[0]
    return L


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    cat = filters.catalog()
    x3 = synth.config3_frame(n)
    cases = [(nm, x3) for nm in ("rp2", "rp4", "rp8", "rp16", "rp32", "rp4_k2", "rp4_k4", "bw6")]
    cases += [("bw48", synth.config5_frame(n)),
              ("rp6", synth.config4_stream(1, n)[0].astype(np.float32)),
              ("rp4", x3[: n - 37, : n - 5])]
    for nm, x in cases:
        f = cat[nm]
        Lref = O.laplacian(O.blur(x, f))
        sc = np.abs(Lref).max()
        e64 = np.abs(lapfirst2d(x, f, np.float64) - Lref).max() / sc
        e32 = np.abs(lapfirst2d(x, f, F).astype(np.float64) - Lref)
        T32 = O.iir_rows(x, f).astype(np.float32).astype(np.float64)
        cur = np.abs(O.laplacian(O.iir_cols(T32, f)) - Lref).max() / sc
        print(f"{nm:7s} {x.shape}: fp64 algebra {e64:.1e}  fp32 {e32.max() / sc:.2e} "
              f"(border rows/cols {max(e32[0].max(), e32[-1].max(), e32[:, 0].max(), e32[:, -1].max()) / sc:.1e})"
              f"  | fp64 rows + fp64 cols on fp32 T: {cur:.2e}", flush=True)
