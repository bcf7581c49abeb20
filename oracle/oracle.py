"""CPU oracle: restatement of the reference hot path -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may use this module.

Numerics come from the C restatement in vmf_oracle.c (fp64, the reference's
operation order, no FMA contraction; bit-identical to the reference's numba
kernels -- pinned by tests/test_oracle.py against tests/golden/).  The
stage-4 detection rule has no reference function; it is restated from
SURVEY.md §8(d) in C (orc_detect3x3*) and, independently, in numpy below
(`detect3x3_np`) so the two restatements check each other.

Function  ->  reference (/root/reference/pkg/src/vmfilt/)
  iir_rows / iir_cols     engine.py:137-158 (kernel 65-102)
  conv_rows / conv_cols   engine.py:112-126 (kernel 35-62)
  blur                    apply_cols(apply_rows(img, s), s)  engine.py:161-174
  laplacian               derivative_field D20 + D02  engine.py:205-228, blob.py:161
  detect3x3 / detect3x3x3 SURVEY.md §8(d) rule (blob.py:162-168 conventions)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "build", "libvmf_oracle.so")
_lib = None
_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        i64 = C.c_int64
        L.orc_iir_rows.argtypes = [_dp, _dp, i64, i64, _dp, _dp, C.c_int, C.c_double, C.c_double]
        L.orc_iir_cols.argtypes = L.orc_iir_rows.argtypes
        L.orc_conv_rows.argtypes = [_dp, _dp, i64, i64, _dp, C.c_int]
        L.orc_conv_cols.argtypes = L.orc_conv_rows.argtypes
        L.orc_laplacian.argtypes = [_dp, _dp, i64, i64]
        L.orc_absmax.argtypes = [_dp, i64]
        L.orc_absmax.restype = C.c_double
        L.orc_detect3x3.argtypes = [_dp, i64, i64, C.c_double, _ip, _ip, _dp, i64]
        L.orc_detect3x3.restype = i64
        L.orc_detect3x3x3.argtypes = [_dp, i64, i64, i64, C.c_double, _ip, _ip, _ip, _dp, i64]
        L.orc_detect3x3x3.restype = i64
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_max_threads.restype = C.c_int
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


def max_threads() -> int:
    return lib().orc_max_threads()


def _img(x) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if a.ndim != 2 or a.shape[0] < 1 or a.shape[1] < 1:
        raise ValueError("image must be a 2-D array")
    return a


def _is_fir(stage):
    return hasattr(stage, "taps")


def _iir(x, f, cols):
    a = _img(x)
    h, w = a.shape
    k = len(f.a_plus)
    if (h if cols else w) < 2 * k + 1:
        raise ValueError("line shorter than 2K+1")
    out = np.empty_like(a)
    bp = np.ascontiguousarray(f.b_plus, dtype=np.float64).reshape(-1)
    ap = np.ascontiguousarray(f.a_plus, dtype=np.float64).reshape(-1)
    if k == 0:
        bp = ap = np.zeros(1)
    sign = 1.0 if f.parity == "sym" else -1.0
    (lib().orc_iir_cols if cols else lib().orc_iir_rows)(a, out, h, w, bp, ap, k,
                                                         float(f.b_zero), sign)
    return out


def _conv(x, kernel, cols):
    a = _img(x)
    h, w = a.shape
    taps = np.ascontiguousarray(kernel.taps, dtype=np.float64)
    if taps.size > (h if cols else w):
        raise ValueError("kernel longer than line")
    out = np.empty_like(a)
    (lib().orc_conv_cols if cols else lib().orc_conv_rows)(a, out, h, w, taps, taps.size)
    return out


def iir_rows(x, f):
    return _iir(x, f, False)


def iir_cols(x, f):
    return _iir(x, f, True)


def conv_rows(x, kernel):
    return _conv(x, kernel, False)


def conv_cols(x, kernel):
    return _conv(x, kernel, True)


def apply_rows(x, stage):
    return conv_rows(x, stage) if _is_fir(stage) else iir_rows(x, stage)


def apply_cols(x, stage):
    return conv_cols(x, stage) if _is_fir(stage) else iir_cols(x, stage)


def blur(x, stage, col_stage=None):
    return apply_cols(apply_rows(x, stage), col_stage if col_stage is not None else stage)


def laplacian(b):
    a = _img(b)
    out = np.empty_like(a)
    lib().orc_laplacian(a, out, a.shape[0], a.shape[1])
    return out


def absmax(a) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(lib().orc_absmax(a.reshape(-1), a.size))


def detect3x3(L, frac=0.5, thr=None):
    """-> (ys, xs, vals, thr), sorted by (y, x)."""
    a = _img(L)
    if thr is None:
        thr = frac * absmax(a)
    cap = a.size
    ys = np.empty(cap, np.int32)
    xs = np.empty(cap, np.int32)
    vs = np.empty(cap, np.float64)
    n = lib().orc_detect3x3(a, a.shape[0], a.shape[1], float(thr), ys, xs, vs, cap)
    return ys[:n], xs[:n], vs[:n], thr


def detect3x3x3(N, frac=0.5, thr=None):
    """-> (ss, ys, xs, vals, thr), sorted by (s, y, x)."""
    a = np.ascontiguousarray(np.asarray(N, dtype=np.float64))
    ns, h, w = a.shape
    if thr is None:
        thr = frac * absmax(a)
    cap = a.size
    ss = np.empty(cap, np.int32)
    ys = np.empty(cap, np.int32)
    xs = np.empty(cap, np.int32)
    vs = np.empty(cap, np.float64)
    n = lib().orc_detect3x3x3(a.reshape(-1), ns, h, w, float(thr), ss, ys, xs, vs, cap)
    return ss[:n], ys[:n], xs[:n], vs[:n], thr


def detect3x3_np(L, frac=0.5, thr=None):
    """Independent numpy restatement of the 3x3 rule (edge padding)."""
    a = np.asarray(L, dtype=np.float64)
    if thr is None:
        thr = frac * np.abs(a).max()
    p = np.pad(a, 1, mode="edge")
    h, w = a.shape
    gt = np.ones_like(a, dtype=bool)
    lt = np.ones_like(a, dtype=bool)
    for di in (-1, 0, 1):
        for dj in (-1, 0, 1):
            if di == 0 and dj == 0:
                continue
            nb = p[1 + di:1 + di + h, 1 + dj:1 + dj + w]
            gt &= a > nb
            lt &= a < nb
    mask = (gt & (a >= thr)) | (lt & (-a >= thr))
    ys, xs = np.nonzero(mask)
    return ys.astype(np.int32), xs.astype(np.int32), a[ys, xs], thr


def pipeline(x, stage, col_stage=None, frac=0.5, lap_scale=1.0):
    """Full hot path: blur -> Laplacian (* lap_scale) -> 3x3 detection."""
    B = blur(x, stage, col_stage)
    L = laplacian(B)
    if lap_scale != 1.0:
        L = L * lap_scale
    return B, L, detect3x3(L, frac)


# ---------------------------------------------------------------------------
# Hessian blob detector (blob.py:109-179)
# ---------------------------------------------------------------------------
_BANK3 = ((0.0, 1.0, 0.0), (0.5, 0.0, -0.5), (1.0, -2.0, 1.0))  # fir_vm_bank(3), design.py:250


class _Taps:
    def __init__(self, taps):
        self.taps = tuple(taps)


def derivative_field(x, stage, order=3, bank=None):
    """engine.derivative_field (engine.py:205-228): blur once, then the
    minimal-support differentiator bank (taps per derivative order; default
    fir_vm_bank(3)), conv_rows for d_x then conv_cols for d_y, each with
    replicate edges; pairs with d_x + d_y >= order skipped."""
    bank = _BANK3 if bank is None else bank
    b = blur(x, stage)
    out = {}
    for dx in range(order):
        for dy in range(order):
            if dx + dy >= order:
                continue
            o = b
            if dx:
                o = conv_rows(o, _Taps(bank[dx]))
            if dy:
                o = conv_cols(o, _Taps(bank[dy]))
            out[(dx, dy)] = o
    return out


def hessian_fields(field, sigma):
    """nd = sigma^4 (D20 D02 - D11^2) (blob.py:109-111), trace D20 + D02, and
    the displacement dx, dy with NaN where |det| < 1e-12 (blob.py:114-128)."""
    d10, d01 = field[(1, 0)], field[(0, 1)]
    d20, d02, d11 = field[(2, 0)], field[(0, 2)], field[(1, 1)]
    nd = sigma ** 4 * (d20 * d02 - d11 ** 2)
    det = d20 * d02 - d11 * d11
    with np.errstate(divide="ignore", invalid="ignore"):
        dx = (d01 * d11 - d02 * d10) / det
        dy = (d10 * d11 - d20 * d01) / det
    bad = np.abs(det) < 1e-12
    dx[bad] = np.nan
    dy[bad] = np.nan
    return nd, d20 + d02, dx, dy


def hessian_detect(x, stage, lam, t1, t2=None, polarity="dark"):
    """blob.detect (blob.py:143-179) with an explicit blur stage: candidates
    nd > t1 with the trace polarity, visited in lexsort((x, y, -nd)) order,
    greedy suppression within (lam/2)^2, then the optional t2 displacement
    filter.  Returns a list of (x, y, dx, dy, nd) tuples, strongest first."""
    if t1 <= 0:
        raise ValueError("t1 must be positive")
    if polarity not in ("dark", "bright"):
        raise ValueError("polarity must be 'dark' or 'bright'")
    sigma = lam / 2.0
    nd, trace, dx, dy = hessian_fields(derivative_field(x, stage, 3), sigma)
    mask = nd > t1
    mask &= (trace > 0) if polarity == "dark" else (trace < 0)
    ys, xs = np.nonzero(mask)
    if ys.size == 0:
        return []
    scores = nd[ys, xs]
    order = np.lexsort((xs, ys, -scores))
    kept = []
    r2 = (lam / 2.0) ** 2
    for i in order:
        xx, yy = int(xs[i]), int(ys[i])
        if any((xx - k[0]) ** 2 + (yy - k[1]) ** 2 <= r2 for k in kept):
            continue
        kept.append((xx, yy, float(dx[yy, xx]), float(dy[yy, xx]), float(nd[yy, xx])))
    if t2 is not None:
        kept = [k for k in kept if np.hypot(k[2], k[3]) <= t2]
    return kept
