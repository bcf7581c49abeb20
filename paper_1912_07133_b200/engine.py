"""Drop-in GPU replacement for the reference's separable filtering engine
(/root/reference/pkg/src/vmfilt/engine.py).

Same names, argument meaning and error behaviour:

=================  ==========================  ===================================
this module        reference (engine.py)       native entry (include/vmfilt_b200.h)
=================  ==========================  ===================================
conv_rows          112-121 (+ kernel 35-62)     vmf_conv_rows
conv_cols          124-126                      vmf_conv_cols
iir_rows           137-153 (+ kernel 65-102)    vmf_iir_rows
iir_cols           156-158                      vmf_iir_cols
apply_rows/cols    161-174                      dispatch on stage type
apply_separable    177-187                      rows then columns
derivative_field   190-228                      blur + vmf_conv_* bank
stability_margin   129-134                      (host, np.roots like the reference)
=================  ==========================  ===================================

Inputs may be numpy arrays / array-likes (returned as numpy float32, with the
host<->device copies done here) or torch tensors (returned as CUDA float32
tensors, no host round trip).  Computation is fp32 in / fp32 out with fp64
recurrence state and fp64 accumulation on the GPU; the reference computes and
returns float64.  There is no CPU fallback: without a CUDA device or the
built library every call raises.
"""
from __future__ import annotations

import ctypes as C
import functools
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import StabilityError
from .filters import is_fir, is_iir

__all__ = [
    "conv_rows", "conv_cols", "iir_rows", "iir_cols", "apply_rows", "apply_cols",
    "SeparableFilter", "apply_separable", "DerivativeField", "derivative_field",
    "stability_margin", "laplacian", "set_threads", "max_threads", "crop_border",
]


# ---------------------------------------------------------------------------
# host <-> device plumbing
# ---------------------------------------------------------------------------
def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("vmfilt-b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _as_image(img):
    """Validate like engine.py:105-109 and stage on the GPU.

    Returns (tensor on device, 'numpy'|'torch', vmf dtype code).  Integer
    samples stay integer and are converted inside the first pass: uint16
    (host order), uint8, and big-endian uint16 (numpy '>u2', e.g. PGM P5
    samples from pgmio.read_pgm_raw; byte-swapped on the GPU).  Everything
    else becomes float32."""
    code = None
    if isinstance(img, torch.Tensor):
        t, kind = img, "torch"
    else:
        a = np.asarray(img)
        if a.dtype == np.dtype(">u2") and a.dtype.byteorder != "=":
            code = _lib.VMF_U16BE
            a = np.ascontiguousarray(a).view(np.uint16)  # the file's bytes, unswapped
        elif a.dtype not in (np.uint16, np.uint8):
            a = np.asarray(a, dtype=np.float32)
        t, kind = torch.from_numpy(np.ascontiguousarray(a)), "numpy"
    if t.ndim != 2 or t.shape[0] < 1 or t.shape[1] < 1:
        raise ValueError("image must be a 2-D array")
    if t.dtype not in (torch.float32, torch.uint16, torch.uint8):
        t = t.to(torch.float32)
    dev = _device()
    if t.device != dev:
        t = t.to(dev, non_blocking=True)
    if t.stride(1) != 1 or t.stride(0) < t.shape[1]:
        t = t.contiguous()
    if code is None:
        code = {torch.uint16: _lib.VMF_U16, torch.uint8: _lib.VMF_U8}.get(t.dtype, _lib.VMF_F32)
    return t, kind, code


def _finish(out: torch.Tensor, kind: str):
    return out.cpu().numpy() if kind == "numpy" else out


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


_ws_cache: dict = {}


def _workspace(nbytes: int, slot: int = 0) -> torch.Tensor:
    """Grow-only scratch buffer per device and slot (caller-owned workspace of
    the C ABI).  Work queued concurrently on different streams uses
    different slots."""
    dev = _device()
    buf = _ws_cache.get((dev, slot))
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(int(nbytes), 1 << 20), dtype=torch.uint8, device=dev)
        _ws_cache[(dev, slot)] = buf
    return buf


def _dptr(vals) -> C.Array:
    arr = (C.c_double * max(len(vals), 1))(*[float(v) for v in vals])
    return arr


def _ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


def _pitch(t: torch.Tensor) -> int:
    """Row pitch in elements (stride of a size-1 dim is arbitrary)."""
    return t.stride(0) if t.shape[0] > 1 else t.shape[1]


# ---------------------------------------------------------------------------
# reference-mirroring host checks
# ---------------------------------------------------------------------------
def stability_margin(f) -> float:
    """1 - max |pole|; positive for a usable recursion (engine.py:129-134)."""
    return _margin(tuple(float(v) for v in f.a_plus))


@functools.lru_cache(maxsize=256)
def _margin(a_plus: tuple) -> float:
    # memoised: the fused paths check both stages on every call
    if len(a_plus) == 0:
        return 1.0
    roots = np.roots(np.concatenate(([1.0], np.asarray(a_plus, dtype=np.float64))))
    return float(1.0 - np.max(np.abs(roots))) if roots.size else 1.0


def _iir_checks(f, length: int) -> None:
    k = len(f.a_plus)
    if k > _lib.MAX_IIR_ORDER:
        raise ValueError(f"IIR order {k} > {_lib.MAX_IIR_ORDER}")
    if length < 2 * k + 1:
        raise ValueError(f"row length {length} < 2K+1 = {2 * k + 1}")
    if stability_margin(f) <= 0.0:
        raise StabilityError("recursion has a pole on or outside the unit circle")


def _fir_checks(kernel, length: int) -> None:
    n = len(kernel.taps)
    if n > length:
        raise ValueError(f"kernel length {n} exceeds row length {length}")


def _sign(f) -> int:
    return 1 if f.parity == "sym" else -1


# ---------------------------------------------------------------------------
# device-level passes on CUDA tensors (no host round trip)
# ---------------------------------------------------------------------------
def _iir_dev(x: torch.Tensor, code: int, f, cols: bool) -> torch.Tensor:
    h, w = x.shape
    _iir_checks(f, h if cols else w)
    k = len(f.a_plus)
    y = torch.empty((h, w), dtype=torch.float32, device=x.device)
    lines, length = (w, h) if cols else (h, w)
    L = _lib.lib()
    nbytes = (L.vmf_iir_cols_workspace_bytes(h, w, k) if cols
              else L.vmf_iir_workspace_bytes(lines, length, k))
    ws = _workspace(nbytes)
    fn = L.vmf_iir_cols if cols else L.vmf_iir_rows
    _lib.check(fn(_ptr(x), code, _ptr(y), h, w, _pitch(x), w, _dptr(f.b_plus),
                  _dptr(f.a_plus), k, float(f.b_zero), _sign(f), _ptr(ws), ws.numel(),
                  _stream()))
    return y


def _fir_dev(x: torch.Tensor, code: int, kernel, cols: bool) -> torch.Tensor:
    h, w = x.shape
    _fir_checks(kernel, h if cols else w)
    y = torch.empty((h, w), dtype=torch.float32, device=x.device)
    L = _lib.lib()
    fn = L.vmf_conv_cols if cols else L.vmf_conv_rows
    _lib.check(fn(_ptr(x), code, _ptr(y), h, w, _pitch(x), w, _dptr(kernel.taps),
                  len(kernel.taps), _stream()))
    return y


def _apply_dev(x, code, stage, cols):
    if is_fir(stage):
        return _fir_dev(x, code, stage, cols)
    if is_iir(stage):
        return _iir_dev(x, code, stage, cols)
    raise TypeError(f"unsupported stage type {type(stage).__name__}")


# ---------------------------------------------------------------------------
# public API (engine.py names)
# ---------------------------------------------------------------------------
def conv_rows(img, kernel):
    x, kind, code = _as_image(img)
    return _finish(_fir_dev(x, code, kernel, False), kind)


def conv_cols(img, kernel):
    x, kind, code = _as_image(img)
    return _finish(_fir_dev(x, code, kernel, True), kind)


def iir_rows(img, f):
    x, kind, code = _as_image(img)
    return _finish(_iir_dev(x, code, f, False), kind)


def iir_cols(img, f):
    x, kind, code = _as_image(img)
    return _finish(_iir_dev(x, code, f, True), kind)


def apply_rows(img, stage):
    if not (is_fir(stage) or is_iir(stage)):
        raise TypeError(f"unsupported stage type {type(stage).__name__}")
    x, kind, code = _as_image(img)
    return _finish(_apply_dev(x, code, stage, False), kind)


def apply_cols(img, stage):
    if not (is_fir(stage) or is_iir(stage)):
        raise TypeError(f"unsupported stage type {type(stage).__name__}")
    x, kind, code = _as_image(img)
    return _finish(_apply_dev(x, code, stage, True), kind)


@dataclass(frozen=True)
class SeparableFilter:
    """A 2-D filter as an x-stage (rows) and a y-stage (columns)
    (engine.py:177-183)."""

    x_stage: object
    y_stage: object
    label: tuple = (0, 0)


def apply_separable(img, f: SeparableFilter):
    x, kind, code = _as_image(img)
    t = _apply_dev(x, code, f.x_stage, False)
    return _finish(_apply_dev(t, _lib.VMF_F32, f.y_stage, True), kind)


@dataclass
class DerivativeField:
    """Bank of smoothed derivative images D[(d_x, d_y)] (engine.py:190-202)."""

    images: dict
    order: int
    sigma: float = 0.0

    def __getitem__(self, key):
        return self.images[key]

    def __contains__(self, key):
        return key in self.images


def derivative_field(img, lpf, order: int = 3, sigma: float = 0.0,
                     keep_all: bool = False) -> DerivativeField:
    """Blur once (rows then columns), then apply the minimal-support
    differentiator bank fir_vm_bank(order) (engine.py:205-228; the bank from
    design.fir_vm_bank, bit-identical to the reference's, so orders 3..9 and
    the reference's ValueError for anything else)."""
    if order % 2 != 1:
        raise ValueError("order must be odd")
    from .design import fir_vm_bank

    bank = fir_vm_bank(order, cascade_mode="behind_blur")
    x, kind, code = _as_image(img)
    h, w = x.shape
    fir_ok = is_fir(lpf) and len(lpf.taps) <= 385 and h >= 4 and w >= 4 \
        and len(lpf.taps) <= min(h, w)
    iir_ok = is_iir(lpf) and 2 <= len(lpf.a_plus) <= 4 and h >= 64 \
        and -(-(-(-h // 32) * 32) // 64) <= 128 and w >= 2 * len(lpf.a_plus) + 1
    if order == 3 and not keep_all and (fir_ok or iir_ok):
        # the whole bank from the fp64 blur: one fused pass for a FIR blur, the
        # fused IIR column pass writing the fp64 blur for an IIR one
        from .detect import _Stage

        stg = _Stage(lpf)
        L = _lib.lib()
        ws = _workspace(L.vmf_hessian_detect_workspace_bytes(h, w, C.byref(stg.s), C.byref(stg.s)))
        outs = [torch.empty((h, w), dtype=torch.float32, device=x.device) for _ in range(6)]
        _lib.check(L.vmf_derivative_field(
            _ptr(x), code, h, w, _pitch(x), C.byref(stg.s), C.byref(stg.s),
            *[_ptr(o) for o in outs], w, _ptr(ws), ws.numel(), _stream()))
        keys = ((0, 0), (1, 0), (0, 1), (2, 0), (0, 2), (1, 1))
        return DerivativeField({k: _finish(o, kind) for k, o in zip(keys, outs)}, order, sigma)
    blurred = _apply_dev(_apply_dev(x, code, lpf, False), _lib.VMF_F32, lpf, True)
    images = {}
    for dx in range(order):
        for dy in range(order):
            if dx + dy >= order and not keep_all:
                continue
            out = blurred
            if dx:
                out = _fir_dev(out, _lib.VMF_F32, bank[dx], False)
            if dy:
                out = _fir_dev(out, _lib.VMF_F32, bank[dy], True)
            images[(dx, dy)] = _finish(out, kind)
    return DerivativeField(images, order, sigma)


def laplacian(blurred, scale: float = 1.0):
    """scale * (D20 + D02) of an already blurred image in one launch
    (engine.py:218-227 + blob.py:161)."""
    b, kind, code = _as_image(blurred)
    if code != _lib.VMF_F32:
        b = b.to(torch.float32)
    h, w = b.shape
    out = torch.empty((h, w), dtype=torch.float32, device=b.device)
    _lib.check(_lib.lib().vmf_laplacian(_ptr(b), _ptr(out), h, w, _pitch(b), w,
                                        float(scale), _stream()))
    return _finish(out, kind)


def set_threads(n: int) -> None:
    """Kept for API compatibility (engine.py:27-28); the GPU path has no
    thread pool and its output does not depend on launch configuration."""


def max_threads() -> int:
    return 1


def crop_border(img, n: int):
    """engine.py:273-278."""
    if n <= 0:
        return img
    if 2 * n >= min(img.shape):
        raise ValueError("crop larger than image")
    return img[n:-n, n:-n]
