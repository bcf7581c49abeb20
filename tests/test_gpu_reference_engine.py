"""GPU mirrors of the reference's engine tests that pin the separable
application semantics (/root/reference/pkg/tests/test_engine.py:153-190):
stage order, the separable outer product through apply_separable /
SeparableFilter, and the derivative field on a quadratic surface.  The
reference runs in float64; the GPU path has fp32 input/output (fp64 state),
so the tolerances are the reference's scaled to fp32 output rounding."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1912_07133_b200 import design, filters as F

pytestmark = pytest.mark.gpu

FP32_REL = 1e-6  # a few fp32 ulps of the output scale


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"


def _rand_image(seed, shape=(16, 24)):
    return np.random.default_rng(seed).standard_normal(shape)


def test_stage_order_is_immaterial():
    # test_engine.py:153-160: rows-then-columns equals columns-then-rows in
    # the interior (FIR half-width plus the recursive border transient)
    from paper_1912_07133_b200 import engine as E

    x = _rand_image(5, (128, 128)).astype(np.float32)
    iir = design.repeated_pole_blur(2.0)
    fir = F.gaussian_fir(1.5, 0, 8)
    a = E.apply_cols(E.apply_rows(x, fir), iir)
    b = E.apply_rows(E.apply_cols(x, iir), fir)
    k = 54
    inner = (slice(k, -k), slice(k, -k))
    scale = np.abs(a).max()
    assert np.abs(a[inner].astype(np.float64) - b[inner]).max() < FP32_REL * scale
    # and each order matches the oracle on the whole frame
    assert np.abs(a - O.apply_cols(O.apply_rows(x, fir), iir)).max() < FP32_REL * scale
    assert np.abs(b - O.apply_rows(O.apply_cols(x, iir), fir)).max() < FP32_REL * scale


def test_separable_outer_product_impulse():
    # test_engine.py:163-176: apply_separable(impulse, SeparableFilter(hx, hy))
    # is the outer product of the two tap vectors around the impulse
    from paper_1912_07133_b200 import engine as E

    n = 33
    x = np.zeros((n, n), np.float32)
    x[n // 2, n // 2] = 1.0
    hx = design.interp_diff(1)
    hy = F.gaussian_fir(1.0, 0, 4)
    sf = E.SeparableFilter(hx, hy, (1, 0))
    y = E.apply_separable(x, sf)
    tx = np.zeros(n)
    tx[n // 2 - hx.k:n // 2 + hx.k + 1] = hx.taps
    ty = np.zeros(n)
    ty[n // 2 - hy.k:n // 2 + hy.k + 1] = hy.taps
    want = np.outer(ty, tx)
    assert y.dtype == np.float32
    assert np.abs(y - want).max() < FP32_REL * np.abs(want).max()
    # torch in, torch out, and an IIR stage on one axis
    yt = E.apply_separable(torch.from_numpy(x).cuda(),
                           E.SeparableFilter(design.repeated_pole_blur(2.0), hy, (0, 0)))
    assert isinstance(yt, torch.Tensor) and yt.is_cuda
    ref = O.apply_cols(O.apply_rows(x, design.repeated_pole_blur(2.0)), hy)
    assert np.abs(yt.cpu().numpy() - ref).max() < FP32_REL * np.abs(ref).max()


def test_derivative_field_on_quadratic_surface():
    # test_engine.py:179-190: exact second derivatives of a quadratic after a
    # unit-DC blur, in the interior
    from paper_1912_07133_b200 import engine as E

    n = 64
    yy, xx = np.mgrid[0:n, 0:n].astype(np.float64)
    img = (0.5 * xx ** 2 - xx * yy + 3.0 * xx).astype(np.float32)
    lpf = F.gaussian_fir(1.5, 0, 8)
    field = E.derivative_field(img, lpf, order=3)
    c = slice(20, n - 20)
    # the surface reaches ~2.2e3 (fp32 ulp ~2.4e-4): second differences of the
    # fp64 blur carry the input's fp32 rounding only (the surface values are
    # exact in fp32), so the reference's 1e-8 becomes ~1e-4 absolute here
    scale = np.abs(img).max()
    tol = 4 * np.finfo(np.float32).eps * scale
    assert np.abs(field[(2, 0)][c, c] - 1.0).max() < tol
    assert np.abs(field[(1, 1)][c, c] + 1.0).max() < tol
    assert np.abs(field[(0, 2)][c, c]).max() < tol
    want_dx = (xx - yy + 3.0)[c, c]
    assert np.abs(field[(1, 0)][c, c] - want_dx).max() < tol
