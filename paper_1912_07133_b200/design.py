"""Host-side IIR blur design, re-derived from scratch.

The reference designs its filters in the z domain with 60-digit mpmath
polynomial algebra (design.py:426-561, three-part split polyz.py:408-556).
Here the same filters are computed without mpmath:

* repeated_pole_blur -- in the time domain.  The impulse response is
  h(m) = c_imp d(m) + sum_k c_k |m|^k p^|m|, p = exp(-1/sigma), k < K.  Its
  frequency-response constraints (design.py:443-477: unit dc gain, vanishing
  even dc derivatives 2..2 l_d, vanishing even Nyquist derivatives
  0..2(l_pi_bar-1)) are moment conditions sum_m m^(2r) (+-1)^m h(m), whose
  one-sided sums are negative-order polylogarithms Li_-n(+-p) (Eulerian
  polynomials).  The (K+1)^2 system is solved in exact rational arithmetic.
  The three-part form then needs no decomposition: A+(z) = (1 - p/z)^K, the
  causal part is h(1..K) convolved with A+, and b_zero = h(0).
* butterworth_blur / butterworth_appendix -- the bilinear-transform zero-phase
  low-pass 1 / (1 + (Omega/wc)^l) (design.py:485-517, 551-561).  Its poles
  are known in closed form (the s-plane roots mapped by z = (2+s)/(2-s)), so
  no polynomial root finding is involved; the numerator split is an exact
  rational solve of N = a0 (B+ A- + b0 A+ A- + B- A+).
* interp_diff / fir_vm_bank -- the moment-matched differentiators
  (design.py:203-280): integer moment systems, solved exactly over the
  rationals (the taps are exact fractions, rounded once).
* colored_sg_blur -- the stopband-noise-minimising symmetric blur
  (design.py:337-403): a Cholesky solve of its Gram system in decimal
  arithmetic at the reference's working precision (40 + 2K digits), 12 s for
  the 385-tap config-5 kernel instead of ~30 s.
* blunt_exponential_blur -- K cascaded (z^-1 + 2 + z)/((1-p/z)(1-pz))
  stages (design.py:520-548), A+ = (1 - p/z)^K directly.

Every result is pinned against the reference's closed forms and printed
coefficients (tests/test_design.py:90-199 of the reference, restated in
tests/test_design.py here) and against the reference-designed catalog
entries (data/catalog.json).
"""
from __future__ import annotations

import cmath
import math
from fractions import Fraction

import numpy as np

from .errors import DecompositionError, DesignError, SplitError
from .filters import FirKernel, ThreePartIIR

__all__ = ["repeated_pole_blur", "butterworth_blur", "butterworth_cutoff",
           "butterworth_appendix", "blunt_exponential_blur", "blunt_exponential_from_pole",
           "three_part_from_poles", "interp_diff", "fir_vm_bank", "colored_sg_blur"]

COND_LIMIT = 1e12        # design.py:37
UNIT_CIRCLE_TOL = 1e-9   # polyz.py:40


# ---------------------------------------------------------------------------
# exact helpers
# ---------------------------------------------------------------------------
def _eulerian(n: int) -> list:
    """Eulerian numbers A(n, i), i = 0 .. n-1."""
    return [sum((-1) ** j * math.comb(n + 1, j) * (i + 1 - j) ** n for j in range(i + 1))
            for i in range(n)]


def _li_neg(n: int, x: Fraction) -> Fraction:
    """sum_{m >= 1} m^n x^m for |x| < 1 (polylogarithm of order -n)."""
    if n == 0:
        return x / (1 - x)
    poly = sum(Fraction(a) * x ** i for i, a in enumerate(_eulerian(n)))
    return x * poly / (1 - x) ** (n + 1)


def _solve_exact(a: list, b: list) -> list:
    """Gaussian elimination over the rationals (a: n x n, b: n)."""
    n = len(b)
    m = [list(row) + [rhs] for row, rhs in zip(a, b)]
    for c in range(n):
        piv = next((r for r in range(c, n) if m[r][c] != 0), None)
        if piv is None:
            raise DesignError("singular constraint matrix")
        m[c], m[piv] = m[piv], m[c]
        for r in range(n):
            if r != c and m[r][c] != 0:
                f = m[r][c] / m[c][c]
                m[r] = [u - f * v for u, v in zip(m[r], m[c])]
    return [m[i][n] / m[i][i] for i in range(n)]


def _cond(a: list) -> float:
    try:
        return float(np.linalg.cond(np.array([[float(v) for v in row] for row in a])))
    except Exception:  # pragma: no cover
        return float("inf")


def _poly_mul(u: list, v: list) -> list:
    out = [0] * (len(u) + len(v) - 1)
    for i, x in enumerate(u):
        for j, y in enumerate(v):
            out[i + j] += x * y
    return out


# ---------------------------------------------------------------------------
# repeated-pole blur (time-domain moment design)
# ---------------------------------------------------------------------------
def repeated_pole_blur(sigma: float, l_d: int = 1, l_pi_bar: int = 2) -> ThreePartIIR:
    """Blur with all K = l_d + l_pi_bar poles at p = exp(-1/sigma): flat to
    order 2 l_d at dc, l_pi_bar zeros of even order at Nyquist
    (repeated_pole_blur, design.py:443-482)."""
    if sigma < 1:
        raise ValueError("sigma must be >= 1")
    if l_d < 1 or l_pi_bar < 0 or l_d + l_pi_bar > 6:
        raise ValueError("need l_d >= 1 and l_d + l_pi_bar <= 6")
    K = l_d + l_pi_bar
    p = Fraction(math.exp(-1.0 / sigma))
    # rows: (moment order 2r, x) with x = p at dc and -p at Nyquist
    rows = [(2 * r, p, 1 if r == 0 else 0) for r in range(l_d + 1)]
    rows += [(2 * r, -p, 0) for r in range(l_pi_bar)]
    A, rhs = [], []
    for n2, x, target in rows:
        # column k: two-sided moment sum_m m^n2 (x/p)^|m| |m|^k p^|m|
        # = 2 Li_-(k+n2)(x), plus the m = 0 term when k = n2 = 0
        row = [(1 if (k == 0 and n2 == 0) else 0) + 2 * _li_neg(k + n2, x) for k in range(K)]
        row.append(Fraction(1 if n2 == 0 else 0))  # unit impulse
        A.append(row)
        rhs.append(Fraction(target))
    cond = _cond(A)
    if not math.isfinite(cond) or cond > COND_LIMIT:
        raise DesignError(f"ill-conditioned constraint matrix (cond ~ {cond:.3g})")
    c = _solve_exact(A, rhs)
    h = [c[K] + c[0]] + [sum(c[k] * Fraction(m) ** k for k in range(K)) * p ** m
                         for m in range(1, K + 1)]
    a = [Fraction(math.comb(K, m)) * (-p) ** m for m in range(K + 1)]  # (1 - p/z)^K
    b = [sum(a[i] * h[m - i] for i in range(m)) for m in range(1, K + 1)]
    return ThreePartIIR(tuple(float(v) for v in b), tuple(float(v) for v in a[1:]),
                        float(h[0]), "sym")


# ---------------------------------------------------------------------------
# generic numerator split for known poles
# ---------------------------------------------------------------------------
def three_part_from_poles(num: list, den: list, poles, parity: str = "sym") -> ThreePartIIR:
    """Three-part form of the symmetric rational H = N/D (coefficients of
    z^-k .. z^k) whose forward poles (|z| < 1, conjugate-closed) are given:
    A+ = prod (1 - z_q/z), D = a0 A+ A-, and N = a0 (B+ A- + b0 A+ A- + B- A+)
    solved exactly for B+ (z^-1..z^-k), b0, B- (z^1..z^k)
    (the split of polyz.py:408-556, with the roots supplied)."""
    if parity not in ("sym", "anti"):
        raise ValueError("parity must be 'sym' or 'anti'")
    k = (len(den) - 1) // 2
    if len(den) != 2 * k + 1 or len(num) != 2 * k + 1:
        raise DecompositionError("numerator and denominator need 2k+1 coefficients")
    poles = list(poles)
    if len(poles) != k:
        raise SplitError(f"{len(poles)} forward poles for half-order {k}")
    for z in poles:
        if abs(abs(z) - 1) <= UNIT_CIRCLE_TOL:
            raise SplitError(f"marginally stable: root at |z| = {abs(z):.12g}")
        if abs(z) >= 1:
            raise SplitError("forward pole outside the unit circle")
    acc = [complex(1.0)]
    for z in poles:
        acc = _poly_mul(acc, [1.0, -z])
    if max(abs(v.imag) for v in acc) > 1e-12 * max(abs(v) for v in acc):
        raise SplitError("forward factor is not real (unpaired complex roots)")
    ap = [Fraction(v.real) for v in acc]          # z^0 .. z^-k
    am = ap                                       # A-(z) = A+(1/z): z^0 .. z^k
    apm = _poly_mul(ap[::-1], am)                 # A+ A-: z^-k .. z^k
    N = [Fraction(float(v)) for v in num]
    D = [Fraction(float(v)) for v in den]
    a0 = D[k] / apm[k]
    scale = max(abs(v) for v in D)
    if any(abs(a0 * apm[i] - D[i]) > Fraction(1, 10 ** 9) * scale for i in range(2 * k + 1)):
        raise SplitError("split recombination mismatch (denominator not symmetric?)")
    n = 2 * k + 1
    M = [[Fraction(0)] * n for _ in range(n)]     # row i <-> z^(i-k)
    for m in range(1, k + 1):                     # beta_m z^-m A-(z): column m-1
        for t in range(k + 1):
            M[t - m + k][m - 1] += a0 * am[t]
    for i in range(n):                            # b0 A+ A-: column k
        M[i][k] += a0 * apm[i]
    for m in range(1, k + 1):                     # gamma_m z^m A+(z): column k+m
        for t in range(k + 1):
            M[m - t + k][k + m] += a0 * ap[t]
    try:
        u = _solve_exact(M, N)
    except DesignError as exc:
        raise DecompositionError("singular three-part system") from exc
    b_plus, b0, b_minus = u[:k], u[k], u[k + 1:]
    sgn = 1 if parity == "sym" else -1
    bscale = max([abs(v) for v in b_plus] + [abs(b0), Fraction(1, 10 ** 300)])
    if any(abs(bm - sgn * bp) > Fraction(1, 10 ** 9) * bscale for bp, bm in zip(b_plus, b_minus)):
        raise DecompositionError("solved parts violate the declared parity")
    if parity == "anti":
        if abs(b0) > Fraction(1, 10 ** 9) * bscale:
            raise DecompositionError("antisymmetric numerator left a central term")
        b0 = Fraction(0)
    return ThreePartIIR(tuple(float(v) for v in b_plus), tuple(float(v) for v in ap[1:]),
                        float(b0), parity)


# ---------------------------------------------------------------------------
# bilinear Butterworth and blunt exponential
# ---------------------------------------------------------------------------
def _binom_poly(c: float, l: int) -> list:
    """(z + c)^l, ascending powers of z."""
    return [math.comb(l, i) * c ** (l - i) for i in range(l + 1)]


def _bilinear_lowpass(wc: float, l: int) -> ThreePartIIR:
    """H = wc^l (z+1)^l / (wc^l (z+1)^l + (-1)^(l/2) 2^l (z-1)^l), centred,
    i.e. 1 / (1 + (Omega/wc)^l) with Omega = 2 tan(w/2) (design.py:485-492)."""
    zp = _binom_poly(1.0, l)
    zm = _binom_poly(-1.0, l)
    sgn = (-1) ** (l // 2)
    num = [wc ** l * v for v in zp]                               # ascending z^0..z^l
    den = [n + sgn * 2.0 ** l * v for n, v in zip(num, zm)]
    # times z^(-l/2): ascending z^0..z^l -> z^-l/2..z^l/2 (same order)
    # s-plane poles: s^l = (-1)^(l/2+1) wc^l; the stable half maps inside
    poles = []
    for q in range(l):
        s = wc * cmath.exp(1j * math.pi * (l / 2 + 1 + 2 * q) / l)
        if s.real < 0:
            poles.append((2 + s) / (2 - s))
    return three_part_from_poles(num, den, poles, "sym")


def butterworth_cutoff(sigma: float) -> float:
    """Half-gain frequency of a Gaussian of scale sigma (design.py:516-517)."""
    return float(math.sqrt(2 * math.log(2)) / sigma)


def butterworth_blur(sigma: float, l_d: int = 1) -> ThreePartIIR:
    """Butterworth low-pass of order 2(l_d+1) at the Gaussian's half-gain
    cutoff (butterworth_tf / butterworth_blur, design.py:495-513)."""
    if sigma < 1:
        raise ValueError("sigma must be >= 1")
    if l_d < 1:
        raise ValueError("l_d must be >= 1")
    return _bilinear_lowpass(butterworth_cutoff(sigma), 2 * (l_d + 1))


def butterworth_appendix(lam: float) -> ThreePartIIR:
    """Sixth-order bilinear Butterworth with cutoff 1/lambda
    (design.py:551-561)."""
    if lam < 1:
        raise ValueError("lambda must be >= 1")
    return _bilinear_lowpass(1.0 / lam, 6)


def blunt_exponential_from_pole(p: float, k: int = 3) -> ThreePartIIR:
    """K cascaded blunted two-sided exponentials with pole p
    (design.py:532-548): H = ((1-p)^2/4)^K (z^-1+2+z)^K / ((1-p/z)(1-pz))^K."""
    if not 0 < p < 1:
        raise ValueError("pole must satisfy 0 < p < 1")
    if not 1 <= k <= 4:
        raise ValueError("K must be in 1..4")
    c0 = ((1 - p) ** 2 / 4) ** k
    num, den = [1.0], [1.0]
    for _ in range(k):
        num = _poly_mul(num, [1.0, 2.0, 1.0])
        den = _poly_mul(den, [-p, 1 + p * p, -p])
    return three_part_from_poles([c0 * v for v in num], den, [p] * k, "sym")


def blunt_exponential_blur(lam: float, k: int = 3) -> ThreePartIIR:
    """blunt_exponential_from_pole(exp(-1/lambda), K) (design.py:520-529)."""
    if lam < 1:
        raise ValueError("lambda must be >= 1")
    return blunt_exponential_from_pole(math.exp(-1.0 / lam), k)


# ---------------------------------------------------------------------------
# moment-matched FIR differentiators
# ---------------------------------------------------------------------------
def _fir_moment_design(d: int, rows, n: int) -> FirKernel:
    """Taps of parity d % 2 on the delay basis z^s +- z^-s, s = k + delta
    (s = 0: the unit impulse), with the moment rows
    sum_m c_m m^l (+-1)^m = d! [l == d at dc] solved exactly
    (_delay_basis / _fir_from_combo, design.py:203-230)."""
    delta = d % 2
    A, rhs = [], []
    for l, at in rows:
        row = []
        for k in range(n):
            s = k + delta
            alt = -1 if (at == "pi" and s % 2) else 1
            if s == 0:
                row.append(Fraction(1 if l == 0 else 0))
            else:  # z^s and the mirrored (-1)^delta z^-s: both give s^l (l of parity delta)
                row.append(Fraction(2 * alt * s ** l))
        A.append(row)
        rhs.append(Fraction(math.factorial(d)) if (l == d and at == "dc") else Fraction(0))
    cond = _cond(A)
    if not math.isfinite(cond) or cond > COND_LIMIT:
        raise DesignError(f"ill-conditioned constraint matrix (cond ~ {cond:.3g})")
    c = _solve_exact(A, rhs)
    kmax = n - 1 + delta
    coef = {0: Fraction(0)}
    for k, ck in enumerate(c):  # coefficient of z^m
        s = k + delta
        if s == 0:
            coef[0] = ck
        else:
            coef[s] = ck
            coef[-s] = -ck if delta else ck
    taps = tuple(float(coef.get(-m, 0)) for m in range(-kmax, kmax + 1))  # h(m) = c_-m
    return FirKernel(taps, "anti" if delta else "sym", d)


def interp_diff(d: int) -> FirKernel:
    """Minimal-support central differentiator of order d, exact on
    polynomials of degree <= d (design.py:233-247)."""
    if not 0 <= d <= 8:
        raise ValueError("d must be in 0..8")
    delta = d % 2
    n = (d - delta) // 2 + 1
    return _fir_moment_design(d, [(delta + 2 * j, "dc") for j in range(n)], n)


def fir_vm_bank(D: int, l_pi_bar: int = 2, cascade_mode: str = "behind_blur"):
    """D differentiators d = 0..D-1 with common vanishing moments
    (design.py:250-280); standalone mode adds l_pi_bar Nyquist rows."""
    if D % 2 != 1 or not 3 <= D <= 9:
        raise ValueError("D must be odd, 3 <= D <= 9")
    if cascade_mode not in ("behind_blur", "standalone"):
        raise ValueError("cascade_mode must be 'behind_blur' or 'standalone'")
    l_d = (D - 1) // 2
    out = []
    for d in range(D):
        delta = d % 2
        l_dc = l_d - delta + 1
        l_pi = 0 if cascade_mode == "behind_blur" else l_pi_bar
        rows = [(delta + 2 * j, "dc") for j in range(l_dc)]
        rows += [(delta + 2 * j, "pi") for j in range(l_pi)]
        out.append(_fir_moment_design(d, rows, l_dc + l_pi))
    return out


# ---------------------------------------------------------------------------
# colored Savitzky-Golay blur (high-precision decimal arithmetic, no mpmath)
# ---------------------------------------------------------------------------
def _dec_pi(ctx_prec: int):
    """pi by Machin's formula, 16 atan(1/5) - 4 atan(1/239), in the current
    decimal context."""
    from decimal import Decimal

    def atan_inv(n: int):
        x = Decimal(1) / n
        x2 = x * x
        term, total, k = x, x, 1
        eps = Decimal(10) ** (-(ctx_prec + 2))
        while True:
            term = -term * x2
            k += 2
            t = term / k
            if abs(t) < eps:
                return total
            total += t

    return 16 * atan_inv(5) - 4 * atan_inv(239)


def _dec_sin(x, pi, ctx_prec: int):
    """sin(x) by the Taylor series after reduction to [-pi, pi]."""
    from decimal import Decimal

    two_pi = 2 * pi
    x = x - two_pi * (x / two_pi).to_integral_value()
    if x > pi:
        x -= two_pi
    elif x < -pi:
        x += two_pi
    x2 = x * x
    term, total, k = x, x, 1
    eps = Decimal(10) ** (-(ctx_prec + 2))
    while abs(term) > eps:
        term = -term * x2 / ((k + 1) * (k + 2))
        k += 2
        total += term
    return total


def colored_sg_blur(sigma: float, l_d: int = 1) -> FirKernel:
    """Symmetric blur of half-width K = ceil(5 sigma) (ceil(7 sigma) for
    l_d = 2) minimising the preserved noise power on [wc, pi], wc = 3 / sigma,
    under unit dc gain and vanishing even moments up to 2 l_d
    (colored_sg_blur, design.py:337-403).

    The stopband Gram matrix S (Toeplitz-plus-Hankel after folding the tap
    symmetry) is numerically singular in double precision, so the
    constrained minimum c = S^-1 F^T (F S^-1 F^T)^-1 e is computed with a
    Cholesky factorisation of S in decimal arithmetic carrying 40 + 2K
    digits (the precision the reference uses), then rounded once."""
    from decimal import Decimal, localcontext

    if sigma < 1:
        raise ValueError("sigma must be >= 1")
    if l_d not in (1, 2):
        raise ValueError("l_d must be 1 or 2")
    k = math.ceil((5 if l_d == 1 else 7) * sigma)
    n, nr = k + 1, l_d + 1
    dps = max(60, 40 + 2 * k)
    with localcontext() as ctx:
        ctx.prec = dps + 10
        pi = _dec_pi(ctx.prec)
        wc = Decimal(3) / Decimal(repr(float(sigma)))
        sb = [(pi - wc) / pi] + [-_dec_sin(wc * j, pi, ctx.prec) / (pi * j)
                                 for j in range(1, 2 * k + 1)]
        # folded Gram matrix: c_0 is the centre tap, c_j (j >= 1) both taps +-j
        S = [[None] * n for _ in range(n)]
        for a in range(n):
            for b in range(a, n):
                if a == 0 and b == 0:
                    v = sb[0]
                elif a == 0:
                    v = 2 * sb[b]
                else:
                    v = 2 * sb[b - a] + 2 * sb[a + b]
                S[a][b] = S[b][a] = v
        # Cholesky S = L L^T (row-oriented)
        L = [[Decimal(0)] * n for _ in range(n)]
        for i in range(n):
            Li = L[i]
            for j in range(i + 1):
                Lj = L[j]
                acc = S[i][j]
                for q in range(j):
                    acc -= Li[q] * Lj[q]
                if i == j:
                    if acc <= 0:
                        raise DesignError("stopband Gram matrix is not positive definite")
                    Li[i] = acc.sqrt()
                else:
                    Li[j] = acc / Lj[j]
        # F^T columns: moment rows sum_m m^(2r) h(m) in folded coordinates
        Ft = [[Decimal(1 if r == 0 else 0)] + [Decimal(2 * j ** (2 * r)) for j in range(1, n)]
              for r in range(nr)]
        Y = []
        for col in Ft:  # S^-1 F^T by forward / back substitution
            z = [Decimal(0)] * n
            for i in range(n):
                acc = col[i]
                Li = L[i]
                for q in range(i):
                    acc -= Li[q] * z[q]
                z[i] = acc / Li[i]
            yv = [Decimal(0)] * n
            for i in range(n - 1, -1, -1):
                acc = z[i]
                for q in range(i + 1, n):
                    acc -= L[q][i] * yv[q]
                yv[i] = acc / L[i][i]
            Y.append(yv)
        M = [[sum((Ft[r][i] * Y[s][i] for i in range(n)), Decimal(0)) for s in range(nr)]
             for r in range(nr)]
        lam = _solve_exact([[Fraction(v) for v in row] for row in M],
                           [Fraction(1)] + [Fraction(0)] * (nr - 1))
        lam = [Decimal(v.numerator) / Decimal(v.denominator) for v in lam]
        c = [sum((Y[s][i] * lam[s] for s in range(nr)), Decimal(0)) for i in range(n)]
        taps = [float(c[abs(m)]) for m in range(-k, k + 1)]
    # re-centre the rounding so the double-precision sum is exactly 1
    taps[k] += 1.0 - (taps[k] + 2 * math.fsum(taps[k + 1:]))
    return FirKernel(tuple(taps), "sym", 0)
