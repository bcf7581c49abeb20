"""Blocked-precision FIR (VERDICT r1 "next" item 7, first step): can the long
FIR blurs run with fp32 products and fp32 partial sums over <= 32-tap
blocks, the block sums accumulated in fp64?  That is the precision a
tensor-core Toeplitz-GEMM FIR (fp32-accumulating MMA over 32-tap K-slices,
fp64 across slices) would have.

numpy emulation of conv_rows / conv_cols (engine.py:35-62: out[n] =
sum_m taps[k+m] x[n-m], replicate edges): each block's products and sums are
rounded to fp32 (a separate multiply and add per tap, so slightly worse than
an FMA), the intermediate T = rows(X) is stored in fp32 as the product path
stores it, B = cols(T) in fp64, L = 5-point Laplacian (replicate) in fp64.
Variants: "tf32" additionally rounds X / T and the taps to a 10-bit mantissa
(the tcgen05 kind::tf32 operand format).

Metric: max|L - L_ref| / max|L_ref| against the oracle (fp64 throughout);
the parity tolerance is 1e-4.  Run: python tools/experiments/fir_blocked_fp32.py [N]
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np

from oracle import oracle as O
from paper_1912_07133_b200 import filters, synth

F = np.float32


def tf32(a):
    """Round fp32 values to tf32 (10 explicit mantissa bits, nearest-even)."""
    b = np.asarray(a, F).view(np.uint32).astype(np.uint64)
    lsb = (b >> 13) & 1
    b = ((b + 0xFFF + lsb) >> 13) << 13
    return b.astype(np.uint32).view(F)


def conv_blocked(x, taps, axis, block=32, operand=None):
    """Replicate-edge FIR along `axis` with fp32 block sums, fp64 across blocks."""
    X = np.moveaxis(np.asarray(x, np.float64), axis, -1)
    n = X.shape[-1]
    k = (len(taps) - 1) // 2
    Xp = np.concatenate([np.repeat(X[..., :1], k, -1), X, np.repeat(X[..., -1:], k, -1)], -1)
    Xp = Xp.astype(F)
    t32 = np.asarray(taps, F)
    if operand is not None:
        Xp, t32 = operand(Xp), operand(t32)
    acc64 = np.zeros(X.shape, np.float64)
    for b0 in range(0, len(taps), block):
        acc = np.zeros(X.shape, F)
        for j in range(b0, min(b0 + block, len(taps))):
            m = j - k  # out[n] += taps[k+m] x[n-m] = taps[j] Xp[n - m + k]
            acc = acc + t32[j] * Xp[..., k - m: k - m + n]
        acc64 += acc.astype(np.float64)
    return np.moveaxis(acc64, -1, axis)


def split3(a):
    """3xTF32 operand split: a = hi + lo, both tf32."""
    hi = tf32(a)
    lo = tf32(np.asarray(a, F) - hi)
    return hi, lo


def valid_3xtf32(a, taps, axis, block=32):
    """'valid' FIR as the 3xTF32 tensor-core product would form it: per tap,
    hi*hi + hi*lo + lo*hi (tf32 operands, fp32 accumulation in 32-tap K
    slices), the slices summed in fp32 (the TMEM accumulator)."""
    A = np.moveaxis(np.asarray(a, F), axis, -1)
    k = (len(taps) - 1) // 2
    n = A.shape[-1] - 2 * k
    th, tl = split3(np.asarray(taps, F))
    Ah, Al = split3(A)
    acc = np.zeros(A.shape[:-1] + (n,), F)
    for j in range(len(taps)):
        m = j - k
        sl = slice(k - m, k - m + n)
        acc = acc + (th[j] * Ah[..., sl] + (th[j] * Al[..., sl] + tl[j] * Ah[..., sl]))
    return np.moveaxis(acc, -1, axis)


def lapfirst_3xtf32(x, f):
    k = (len(f.taps) - 1) // 2
    P = k + 1
    Xe = np.pad(np.asarray(x, F), P, mode="edge")
    U = ((Xe[1:-1, :-2] - Xe[1:-1, 1:-1]) + (Xe[1:-1, 2:] - Xe[1:-1, 1:-1])) + \
        ((Xe[:-2, 1:-1] - Xe[1:-1, 1:-1]) + (Xe[2:, 1:-1] - Xe[1:-1, 1:-1]))
    V = valid_3xtf32(U, f.taps, 1).astype(F)
    return valid_3xtf32(V, f.taps, 0).astype(np.float64)


def valid_blocked(a, taps, axis, block=32):
    """'valid' FIR along `axis` (no edge rule), fp32 block sums, fp64 across."""
    A = np.moveaxis(np.asarray(a, F), axis, -1)
    k = (len(taps) - 1) // 2
    n = A.shape[-1] - 2 * k
    t32 = np.asarray(taps, F)
    acc64 = np.zeros(A.shape[:-1] + (n,), np.float64)
    for b0 in range(0, len(taps), block):
        acc = np.zeros(acc64.shape, F)
        for j in range(b0, min(b0 + block, len(taps))):
            m = j - k
            acc = acc + t32[j] * A[..., k - m: k - m + n]
        acc64 += acc.astype(np.float64)
    return np.moveaxis(acc64, -1, axis)


def lapfirst_blocked(x, f, block=32, operand=None):
    """Laplacian first (DESIGN.md §2's identity, applied to the FIR): the
    blocked fp32 FIRs run on U = Lap5 of the replicate-extended frame, so
    their rounding is relative to |L|.  Interior pixels only (the four border
    terms are separate fp64-sized corrections)."""
    k = (len(f.taps) - 1) // 2
    P = k + 1
    Xe = np.pad(np.asarray(x, F), P, mode="edge")
    U = ((Xe[1:-1, :-2] - Xe[1:-1, 1:-1]) + (Xe[1:-1, 2:] - Xe[1:-1, 1:-1])) + \
        ((Xe[:-2, 1:-1] - Xe[1:-1, 1:-1]) + (Xe[2:, 1:-1] - Xe[1:-1, 1:-1]))  # fp32, pad k
    op = operand or (lambda a: a)
    V = valid_blocked(op(U), op(np.asarray(f.taps, F)), 1, block).astype(F)  # stored fp32
    return valid_blocked(op(V), op(np.asarray(f.taps, F)), 0, block)


def lap_blocked(x, f, operand=None, block=32):
    T = conv_blocked(x, f.taps, 1, block, operand).astype(F)  # stored fp32
    B = conv_blocked(T, f.taps, 0, block, operand)
    return O.laplacian(B)


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    cat = filters.catalog()
    cases = [("g8_k32", synth.config3_frame(n)), ("g16_k64", synth.config3_frame(n)),
             ("g32_k128", synth.config3_frame(n)), ("sg38.4", synth.config5_frame(n))]
    for nm, x in cases:
        f = cat[nm]
        Lref = O.laplacian(O.blur(x, f))
        s = np.abs(Lref).max()
        row = [f"{nm:9s} {len(f.taps):3d} taps"]
        for label, op, blk in (("fp32/32", None, 32), ("fp32/8", None, 8), ("tf32/32", tf32, 32)):
            e = np.abs(lap_blocked(x, f, op, blk) - Lref).max() / s
            row.append(f"{label} {e:.2e}")
        # the share of T's fp32 storage alone (fp64 sums, T rounded once)
        T = O.conv_rows(x, f).astype(F).astype(np.float64)
        e = np.abs(O.laplacian(O.conv_cols(T, f)) - Lref).max() / s
        row.append(f"T-store-only {e:.2e}")
        Lf = lapfirst_blocked(x, f)
        e = np.abs(Lf - Lref)[1:-1, 1:-1].max() / s
        row.append(f"lapfirst fp32/32 (interior) {e:.2e}")
        e = np.abs(lapfirst_blocked(x, f, 1 << 20) - Lref)[1:-1, 1:-1].max() / s
        row.append(f"lapfirst fp32/all {e:.2e}")
        e = np.abs(lapfirst_blocked(x, f, 32, tf32) - Lref)[1:-1, 1:-1].max() / s
        row.append(f"lapfirst tf32/32 {e:.2e}")
        e = np.abs(lapfirst_3xtf32(x, f) - Lref)[1:-1, 1:-1].max() / s
        row.append(f"lapfirst 3xtf32 {e:.2e}")
        print("  ".join(row), flush=True)
