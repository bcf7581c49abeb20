"""ctypes binding of libvmfilt_b200.so (the C ABI in include/vmfilt_b200.h).

The shared library is built in-tree by ``make -C paper_1912_07133_b200/csrc``
(or ``__graft_entry__.build()``).  There is no CPU fallback: if the library
is missing every call raises, loudly.
"""
from __future__ import annotations

import ctypes as C
import os

from .errors import StabilityError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libvmfilt_b200.so")
if os.environ.get("VMF_LIB_PATH"):  # A/B builds for experiments (tools/scratch)
    LIB_PATH = os.environ["VMF_LIB_PATH"]

VMF_OK, VMF_EVALUE, VMF_ESTABILITY, VMF_ECUDA = 0, 2, 3, 4
VMF_F32, VMF_U16, VMF_U8, VMF_U16BE = 0, 1, 2, 3
VMF_STAGE_FIR, VMF_STAGE_IIR = 0, 1
MAX_IIR_ORDER = 8
MAX_FIR_TAPS = 2049

_vp, _i64, _sz, _dp = C.c_void_p, C.c_int64, C.c_size_t, C.POINTER(C.c_double)


class VmfStage(C.Structure):
    """struct vmf_stage (include/vmfilt_b200.h)."""

    _fields_ = [
        ("kind", C.c_int),
        ("n", C.c_int),
        ("taps", _dp),
        ("b_plus", _dp),
        ("a_plus", _dp),
        ("b_zero", C.c_double),
        ("sign", C.c_int),
    ]


# name -> (restype, argtypes)
_PROTOS = {
    "vmf_last_error": (C.c_char_p, []),
    "vmf_abi_version": (C.c_int, []),
    "vmf_iir_workspace_bytes": (_sz, [_i64, _i64, C.c_int]),
    "vmf_iir_cols_workspace_bytes": (_sz, [_i64, _i64, C.c_int]),
    "vmf_iir_rows": (C.c_int, [_vp, C.c_int, _vp, _i64, _i64, _i64, _i64, _dp, _dp, C.c_int,
                               C.c_double, C.c_int, _vp, _sz, _vp]),
    "vmf_iir_cols": (C.c_int, [_vp, C.c_int, _vp, _i64, _i64, _i64, _i64, _dp, _dp, C.c_int,
                               C.c_double, C.c_int, _vp, _sz, _vp]),
    "vmf_conv_rows": (C.c_int, [_vp, C.c_int, _vp, _i64, _i64, _i64, _i64, _dp, C.c_int, _vp]),
    "vmf_conv_cols": (C.c_int, [_vp, C.c_int, _vp, _i64, _i64, _i64, _i64, _dp, C.c_int, _vp]),
    "vmf_laplacian": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _i64, C.c_float, _vp]),
    "vmf_detect_workspace_bytes": (_sz, [_i64, _i64]),
    "vmf_detect3x3": (C.c_int, [_vp, _i64, _i64, _i64, C.c_float, _vp, _vp, _i64, _vp, _vp,
                                _vp, _vp, _sz, _vp]),
    "vmf_detect3x3x3_workspace_bytes": (_sz, [_i64, _i64, _i64]),
    "vmf_detect3x3x3": (C.c_int, [_vp, _i64, _i64, _i64, _i64, _i64, C.c_float, _vp, _vp,
                                  _i64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "vmf_detect3x3x3_cands": (C.c_int, [_vp, _i64, _i64, _i64, _i64, _i64, _vp, _vp, _i64, _vp,
                                        _vp, _vp, _i64, _vp, _vp, _vp]),
    "vmf_detect3x3x3_absmax": (C.c_int, [_vp, _i64, _i64, _i64, _i64, _i64, C.c_float, _vp,
                                         _vp, _vp, _i64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "vmf_launch_count": (C.c_longlong, []),
    "vmf_num_kernel_ids": (C.c_int, []),
    "vmf_kernel_name": (C.c_char_p, [C.c_int]),
    "vmf_profile_begin": (None, []),
    "vmf_profile_stop": (None, []),
    "vmf_profile_read": (C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_longlong), C.c_int]),
    "vmf_profile_end": (C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_longlong), C.c_int]),
    "vmf_profile_timeline": (C.c_int, [C.POINTER(C.c_int), C.POINTER(C.c_float),
                                       C.POINTER(C.c_float), C.c_int]),
    "vmf_blur_lap_detect_workspace_bytes": (_sz, [_i64, _i64, C.POINTER(VmfStage),
                                                  C.POINTER(VmfStage)]),
    "vmf_blur_lap_detect": (C.c_int, [_vp, C.c_int, _i64, _i64, _i64, C.POINTER(VmfStage),
                                      C.POINTER(VmfStage), C.c_float, C.c_float, _vp, _vp, _vp,
                                      _vp, _i64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "vmf_sweep_workspace_bytes": (_sz, [_i64, _i64, C.c_int]),
    "vmf_sweep_detect_workspace_bytes": (_sz, [_i64, _i64, C.POINTER(VmfStage)]),
    "vmf_sweep_supported": (C.c_int, [_vp, C.c_int, _i64, _i64, _i64, C.c_int,
                                      C.POINTER(VmfStage), C.POINTER(VmfStage)]),
    "vmf_sweep_rows": (C.c_int, [_vp, C.c_int, _i64, _i64, _i64, C.c_int, C.POINTER(VmfStage),
                                 C.POINTER(VmfStage), _vp, _sz, _vp]),
    "vmf_sweep_detect": (C.c_int, [C.c_int, _i64, _i64, C.c_int, C.POINTER(VmfStage),
                                   C.c_float, C.c_float, _vp, _vp, _vp, _i64, _vp, _vp, _vp,
                                   _sz, _vp, _sz, _vp]),
    "vmf_hessian_detect_workspace_bytes": (_sz, [_i64, _i64, C.POINTER(VmfStage),
                                                 C.POINTER(VmfStage)]),
    "vmf_hessian_detect": (C.c_int, [_vp, C.c_int, _i64, _i64, _i64, C.POINTER(VmfStage),
                                     C.POINTER(VmfStage), C.c_double, C.c_double, C.c_int, _vp,
                                     _vp, _i64, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _sz,
                                     _vp]),
    "vmf_derivative_field": (C.c_int, [_vp, C.c_int, _i64, _i64, _i64, C.POINTER(VmfStage),
                                       C.POINTER(VmfStage), _vp, _vp, _vp, _vp, _vp, _vp, _i64,
                                       _vp, _sz, _vp]),
    "vmf_greedy_nms_workspace_bytes": (_sz, [_i64, _i64, _i64, C.c_double]),
    "vmf_greedy_nms": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _i64, C.c_double, _vp, _vp, _vp,
                                 _sz, _vp]),
}

_lib = None


def exported_symbols():
    return tuple(_PROTOS)


def lib():
    """Load (once) and return the CDLL; raises if the build is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `make -C {_HERE}/csrc` "
                "(there is no CPU fallback)")
        handle = C.CDLL(LIB_PATH)
        for name, (res, args) in _PROTOS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(rc: int) -> None:
    """Map a C-ABI status to the reference's exception types
    (engine.py:115-118,139-142; errors.py:32)."""
    if rc == VMF_OK:
        return
    msg = lib().vmf_last_error().decode(errors="replace")
    if rc == VMF_EVALUE:
        raise ValueError(msg)
    if rc == VMF_ESTABILITY:
        raise StabilityError(msg)
    raise RuntimeError(f"CUDA failure: {msg}")


def launch_count() -> int:
    return int(lib().vmf_launch_count())


def profile_begin() -> None:
    lib().vmf_profile_begin()


def profile_stop() -> None:
    lib().vmf_profile_stop()


def profile_read() -> dict:
    """-> {kernel name: (total_ms, launches)} of the recorded launches."""
    L = lib()
    n = L.vmf_num_kernel_ids()
    ms = (C.c_double * n)()
    cnt = (C.c_longlong * n)()
    L.vmf_profile_read(ms, cnt, n)
    return {L.vmf_kernel_name(i).decode(): (ms[i], cnt[i]) for i in range(n) if cnt[i]}


def profile_timeline(n: int = 4096) -> list:
    """-> [(kernel name, start_ms, end_ms)] of the recorded launches, times
    after the first recorded start."""
    L = lib()
    ids = (C.c_int * n)()
    t0 = (C.c_float * n)()
    t1 = (C.c_float * n)()
    m = L.vmf_profile_timeline(ids, t0, t1, n)
    return [(L.vmf_kernel_name(ids[i]).decode(), t0[i], t1[i]) for i in range(m)]


def profile_end() -> dict:
    """-> {kernel name: (total_ms, launches)} for kernels that ran."""
    L = lib()
    n = L.vmf_num_kernel_ids()
    ms = (C.c_double * n)()
    cnt = (C.c_longlong * n)()
    L.vmf_profile_end(ms, cnt, n)
    return {L.vmf_kernel_name(i).decode(): (ms[i], cnt[i]) for i in range(n) if cnt[i]}
