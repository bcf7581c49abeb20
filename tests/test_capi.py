"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/vmfilt_b200.h declares, and its host-side validation mirrors the
reference wrappers (engine.py:105-109, 115-118, 139-142) -- status codes are
returned before anything touches the device."""
import ctypes as C
import os
import re

import pytest

from paper_1912_07133_b200 import _lib

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                   "vmfilt_b200.h")


def _declared():
    src = open(HDR).read()
    return sorted(set(re.findall(r"\b(vmf_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    names = _declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(L, n), n
    assert set(names) <= set(_lib.exported_symbols())


def test_abi_version_and_error_string():
    L = _lib.lib()
    assert L.vmf_abi_version() == 1
    assert isinstance(L.vmf_last_error(), bytes)


def _d(vals):
    return (C.c_double * max(len(vals), 1))(*vals)


def test_iir_validation_codes_without_gpu():
    L = _lib.lib()
    rp4 = ((0.0883, -0.1262, 0.0428), (-2.3364, 1.8196, -0.4724))
    # row shorter than 2K+1 -> VMF_EVALUE (engine.py:139-140)
    rc = L.vmf_iir_rows(None, 0, None, 4, 6, 6, 6, _d(rp4[0]), _d(rp4[1]), 3, 0.09, 1, None, 0,
                        None)
    assert rc == _lib.VMF_EVALUE
    assert b"2K+1" in L.vmf_last_error()
    # pole outside the unit circle -> VMF_ESTABILITY (engine.py:141-142)
    rc = L.vmf_iir_rows(None, 0, None, 4, 16, 16, 16, _d([0.5]), _d([-1.5]), 1, 0.2, 1, None, 0,
                        None)
    assert rc == _lib.VMF_ESTABILITY
    # non-2-D image -> VMF_EVALUE (engine.py:105-109)
    rc = L.vmf_iir_cols(None, 0, None, 0, 16, 16, 16, _d(rp4[0]), _d(rp4[1]), 3, 0.09, 1, None,
                        0, None)
    assert rc == _lib.VMF_EVALUE


def test_fir_validation_codes_without_gpu():
    L = _lib.lib()
    taps = _d([0.25, 0.5, 0.25])
    assert L.vmf_conv_rows(None, 0, None, 4, 2, 2, 2, taps, 3, None) == _lib.VMF_EVALUE  # > w
    assert L.vmf_conv_cols(None, 0, None, 2, 4, 4, 4, taps, 3, None) == _lib.VMF_EVALUE  # > h
    assert L.vmf_conv_rows(None, 0, None, 4, 8, 8, 8, _d([1, 1]), 2, None) == _lib.VMF_EVALUE


def test_python_checks_mirror_reference():
    from paper_1912_07133_b200 import filters as F
    from paper_1912_07133_b200.engine import _iir_checks, stability_margin
    from paper_1912_07133_b200.errors import StabilityError

    bad = F.ThreePartIIR((0.5,), (-1.5,), 0.2, "sym")
    assert stability_margin(bad) < 0
    with pytest.raises(StabilityError):
        _iir_checks(bad, 16)
    with pytest.raises(ValueError):
        _iir_checks(F.get("rp4"), 6)
