"""Row pass in fp32 as T = X - Q(D2 X) ("second-difference form").

For a symmetric blur R with unit DC gain, I - R has a double zero at z = 1,
so I - R = (1 - z^-1)(1 - z) Q(z) with Q stable; on the replicate-extended
row the second difference D = X(n+1) - 2X(n) + X(n-1) is zero outside the
row, hence exactly
    T = R X = X - Q(D)      (zero-state recursions, no edge terms).
Q has the same poles as R: with the modal form of R's causal part
h(m) = c A^(m-1) b, Q's is q(m) = c_q A^(m-1) b, c_q = -c A (A - I)^-2, and
q(0) follows from the difference equation at n = 0.  Q(D) ~ T - X is small,
so fp32 rounding inside the recursion is relative to |T - X|; T keeps one
fp32 rounding of |T| (what the fp64 row pass stores anyway).

Measured: L error (after an fp64 column pass + Laplacian) vs the oracle."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np

from oracle import oracle as O
from paper_1912_07133_b200 import filters, synth

sys.path.insert(0, os.path.dirname(__file__))
from col_lapfirst_chunked import modal  # noqa: E402

F = np.float32


def q_form(f):
    A, b, c = modal(f)
    k = len(b)
    I = np.eye(k)
    AmI = A - I
    cq = -c @ A @ np.linalg.inv(AmI @ AmI)
    q = lambda m: cq @ np.linalg.matrix_power(A, m - 1) @ b
    # n = 0 equation: 2 q(1) - 2 q(0) = 1 - b0
    q0 = q(1) - 0.5 * (1.0 - f.b_zero)
    return A, b, cq, q0, c


def check_q(f, n=400):
    """q must satisfy q(n+1) - 2 q(n) + q(n-1) = -(r(n) - delta(n)) for all n."""
    A, b, cq, q0, c = q_form(f)
    h = [0.0] + [c @ np.linalg.matrix_power(A, m - 1) @ b for m in range(1, n + 2)]
    qq = [q0] + [cq @ np.linalg.matrix_power(A, m - 1) @ b for m in range(1, n + 2)]
    err = 0.0
    for m in range(0, n):
        lhs = qq[m + 1] - 2 * qq[m] + (qq[m - 1] if m > 0 else qq[1])
        rhs = -((h[m] if m > 0 else f.b_zero) - (1.0 if m == 0 else 0.0))
        err = max(err, abs(lhs - rhs))
    return err


def rows_qform32(x, f):
    A, b, cq, q0, _ = q_form(f)
    A32, b32, cq32 = A.astype(F), b.astype(F), cq.astype(F)
    X = x.astype(F)
    Xl = np.hstack([X[:, :1], X[:, :-1]])
    Xr = np.hstack([X[:, 1:], X[:, -1:]])
    D = (Xl - X) + (Xr - X)
    Hh, W = X.shape
    k = len(b)
    yp = np.zeros_like(X)
    ym = np.zeros_like(X)
    u = np.zeros((k, Hh), F)
    for n in range(W):
        yp[:, n] = cq32 @ u
        u = A32 @ u + b32[:, None] * D[:, n]
    u = np.zeros((k, Hh), F)
    for n in range(W - 1, -1, -1):
        ym[:, n] = cq32 @ u
        u = A32 @ u + b32[:, None] * D[:, n]
    Qd = F(q0) * D + yp + ym
    return X - Qd


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    cat = filters.catalog()
    x3 = synth.config3_frame(n)
    cases = [(nm, x3) for nm in ("rp2", "rp4", "rp8", "rp16", "rp32", "rp4_k2", "rp4_k4", "bw6")]
    cases += [("bw48", synth.config5_frame(n)),
              ("rp6", synth.config4_stream(1, n)[0].astype(np.float32))]
    for nm, x in cases:
        f = cat[nm]
        Tref = O.iir_rows(x, f)
        Lref = O.laplacian(O.iir_cols(Tref, f))
        s = np.abs(Lref).max()
        T32 = rows_qform32(x, f)
        eT = np.abs(T32 - Tref).max() / np.abs(Tref).max()
        L = O.laplacian(O.iir_cols(T32.astype(np.float64), f))
        Lr = O.laplacian(O.iir_cols(Tref.astype(np.float32).astype(np.float64), f))
        print(f"{nm:7s} q-eq residual {check_q(f):.1e}  T err/max|T| {eT:.2e}  "
              f"L err {np.abs(L - Lref).max() / s:.2e} (fp64 row pass rounded: "
              f"{np.abs(Lr - Lref).max() / s:.2e})", flush=True)
