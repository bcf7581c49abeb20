"""Coefficient carriers for the hot path.

The reference's stage objects are ``FirKernel`` (design.py:40-77) and
``ThreePartIIR`` (polyz.py:348-405).  The engine here dispatches by duck
typing (``.taps`` -> FIR, ``.a_plus``/``.b_plus`` -> IIR), so objects built
by the reference's own design code are accepted unchanged; the two light
classes below mirror their fields and validation for users without the
reference installed.

``catalog()`` returns the filters of the five BASELINE configs, designed by
the reference's design code (tools/make_catalog.py) and stored as JSON, so the
GPU box needs neither the reference nor mpmath.  ``gaussian_fir`` is a
restatement of design.py:297-334 (float arithmetic only, no linear algebra).
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass
from functools import lru_cache

_DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "catalog.json")

# fir_vm_bank(3, "behind_blur") taps (design.py:250-280); bank[2] = (1,-2,1)
# is pinned by the reference's tests/test_cli.py:41-48.
VM_BANK3 = ((0.0, 1.0, 0.0), (0.5, 0.0, -0.5), (1.0, -2.0, 1.0))
LAPLACIAN_TAPS = VM_BANK3[2]


@dataclass(frozen=True)
class ThreePartIIR:
    """y+(n) = sum b_plus[m] x(n-m) - sum a_plus[m] y+(n-m);
    y-(n) mirrored with b_minus = +/- b_plus; y = y+ + b_zero x + y-
    (polyz.py:350-358)."""

    b_plus: tuple
    a_plus: tuple
    b_zero: float
    parity: str = "sym"

    def __post_init__(self):
        if self.parity not in ("sym", "anti"):
            raise ValueError("parity must be 'sym' or 'anti'")
        if len(self.b_plus) != len(self.a_plus):
            raise ValueError("b_plus and a_plus must have equal length")
        object.__setattr__(self, "b_plus", tuple(float(v) for v in self.b_plus))
        object.__setattr__(self, "a_plus", tuple(float(v) for v in self.a_plus))
        object.__setattr__(self, "b_zero", float(self.b_zero))
        if self.parity == "anti" and self.b_zero != 0.0:
            raise ValueError("antisymmetric filters must have b_zero = 0")

    @property
    def k(self) -> int:
        return len(self.a_plus)

    @property
    def b_minus(self) -> tuple:
        return self.b_plus if self.parity == "sym" else tuple(-v for v in self.b_plus)

    @property
    def a_minus(self) -> tuple:
        return self.a_plus


@dataclass(frozen=True)
class FirKernel:
    """Centred taps h(-K..K) (design.py:40-77)."""

    taps: tuple
    parity: str = "sym"
    d: int = 0

    def __post_init__(self):
        object.__setattr__(self, "taps", tuple(float(t) for t in self.taps))
        if len(self.taps) % 2 != 1:
            raise ValueError("taps must have odd length 2K+1")
        if self.parity not in ("sym", "anti"):
            raise ValueError("parity must be 'sym' or 'anti'")
        k = self.k
        scale = max(abs(t) for t in self.taps) or 1.0
        sgn = 1.0 if self.parity == "sym" else -1.0
        for m in range(1, k + 1):
            if abs(self.taps[k - m] - sgn * self.taps[k + m]) > 1e-12 * scale:
                raise ValueError(f"taps violate declared parity '{self.parity}'")
        if self.parity == "anti" and abs(self.taps[k]) > 1e-12 * scale:
            raise ValueError("antisymmetric kernel must have zero center tap")
        if self.d == 0 and abs(sum(self.taps) - 1.0) > 1e-12:
            raise ValueError("blur kernel (d=0) must sum to 1")

    @property
    def k(self) -> int:
        return (len(self.taps) - 1) // 2


def is_fir(stage) -> bool:
    return hasattr(stage, "taps")


def is_iir(stage) -> bool:
    return hasattr(stage, "a_plus") and hasattr(stage, "b_plus")


def gaussian_fir(sigma: float, d: int, k: int) -> FirKernel:
    """Windowed sampled Gaussian derivative renormalised to unit dc blur gain
    (restates design.py:297-334; TruncationError -> ValueError here)."""
    if sigma <= 0:
        raise ValueError("sigma must be positive")
    if d < 0:
        raise ValueError("d must be >= 0")
    if k < math.ceil(3 * sigma):
        raise ValueError("K must be at least ceil(3*sigma)")
    sigma2 = sigma * sigma
    norm = 1.0 / (math.sqrt(2 * math.pi) * sigma)

    def g0(m):
        return norm * math.exp(-m * m / (2 * sigma2))

    far = max(k + 1, math.ceil(12 * sigma))
    full = g0(0) + 2 * sum(g0(m) for m in range(1, far + 1))
    win = g0(0) + 2 * sum(g0(m) for m in range(1, k + 1))
    if 1.0 - win / full > 1e-3:
        raise ValueError(f"window K={k} leaves tail mass > 1e-3 for sigma={sigma}")
    c_g = 1.0 / win
    p = [1.0]
    for _ in range(d):  # p_{k+1} = x p_k - sigma^2 p_k'  (design.py:283-294)
        nxt = [0.0] * (len(p) + 1)
        for i, ci in enumerate(p):
            nxt[i + 1] += ci
            if i >= 1:
                nxt[i - 1] -= sigma2 * i * ci
        p = nxt
    sgn = (-1.0) ** d / sigma2 ** d
    taps = []
    for m in range(-k, k + 1):
        pm = 0.0
        for i in reversed(range(len(p))):
            pm = pm * m + p[i]
        taps.append(c_g * sgn * pm * g0(m))
    return FirKernel(tuple(taps), "anti" if d % 2 else "sym", d)


@lru_cache(maxsize=1)
def _catalog_raw() -> dict:
    with open(_DATA) as fh:
        return json.load(fh)


def catalog() -> dict:
    """name -> ThreePartIIR | FirKernel for every designed filter shipped."""
    out = {}
    for name, e in _catalog_raw().items():
        if e["type"] == "iir":
            out[name] = ThreePartIIR(tuple(e["b_plus"]), tuple(e["a_plus"]), e["b_zero"],
                                     e["parity"])
        else:
            out[name] = FirKernel(tuple(e["taps"]), e["parity"], e["d"])
    return out


def get(name: str):
    return catalog()[name]


def design_call(name: str) -> str:
    """The reference design call that produced catalog entry `name`."""
    return _catalog_raw()[name]["design"]
