"""The tensor-core FIR path (vmf_firtc.cu: both FIR passes as banded
Toeplitz products on tcgen05, 3xTF32, Laplacian first) against the oracle
restatement of engine.py:35-62 / 205-228 and stage 4.  Kernels shorter than
kFirTcMinTaps take the fp64 CUDA-core path by default; VMF_FORCE_FIRTC routes
them here so every tap length, shape and edge case runs on the tensor cores.
Each test also checks that the tensor-core kernels actually launched."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1912_07133_b200 import filters as F
from tests.parity import TOL_REL, compare_blobs, max_rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _force_tc(monkeypatch):
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    monkeypatch.setenv("VMF_FORCE_FIRTC", "1")


class _Taps:  # any taps (no parity / sum checks): the C ABI takes them as given
    def __init__(self, taps):
        self.taps = tuple(float(t) for t in taps)


def _frame(h, w, seed, nblobs=8, noise=0.05):
    rng = np.random.default_rng(seed)
    x = (noise * rng.standard_normal((h, w))).astype(np.float32)
    yy, xx = np.ogrid[:h, :w]
    for _ in range(nblobs):
        cy, cx = rng.integers(0, h), rng.integers(0, w)
        x += np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / 18.0).astype(np.float32)
    return x


def _run(x, stage, col_stage=None, frac=0.5, lap_scale=1.0):
    from paper_1912_07133_b200 import _lib, detect

    _lib.profile_begin()
    dets, blur, lap = detect.blur_laplacian_detect(x, stage, frac=frac, col_stage=col_stage,
                                                   lap_scale=lap_scale, return_fields=True)
    torch.cuda.synchronize()
    _lib.profile_stop()
    prof = _lib.profile_read()
    assert "firtc_rows" in prof and "firtc_cols" in prof, sorted(prof)
    B, L, (ys, xs, vs, thr) = O.pipeline(x, stage, col_stage, frac=frac, lap_scale=lap_scale)
    el = max_rel_err(lap, L)
    assert el < TOL_REL, ("laplacian", el)
    assert max_rel_err(blur, B) < TOL_REL
    exempt, bad = compare_blobs(dets.as_set(), set(zip(ys.tolist(), xs.tolist())), L, thr)
    assert not bad, bad[:10]
    assert not dets.overflow
    return el, dets.count, len(ys)


@pytest.mark.parametrize("name,shape", [
    ("g2_k8", (512, 512)), ("g4_k16", (257, 388)), ("g8_k32", (300, 516)),
    ("g16_k64", (1000, 1032)), ("g32_k128", (640, 700)), ("sg38.4", (600, 800)),
    ("sg3.2", (129, 132)),
])
def test_firtc_matches_oracle(cat, name, shape):
    """Catalog FIR kernels over shapes that are and are not multiples of the
    128-sample tiles (partial tiles on both axes, lines H .. H+3 of the row
    pass in a tile of their own or sharing one)."""
    el, n_gpu, n_ref = _run(_frame(*shape, seed=shape[0] * 7 + shape[1]), cat[name])
    assert el < 2e-5


def test_firtc_antisymmetric_and_asymmetric_taps():
    """The border terms use the causal taps t[k+m] on the right / bottom and
    the anticausal t[k-m] on the left / top: an antisymmetric (derivative)
    kernel and a kernel with no symmetry at all."""
    rng = np.random.default_rng(3)
    half = rng.uniform(0.1, 1.0, 12)
    anti = F.FirKernel(tuple(np.concatenate([-half[::-1], [0.0], half]).tolist()), "anti", 1)
    _run(_frame(300, 400, 1), anti)
    taps = rng.uniform(-0.2, 1.0, 41)
    _run(_frame(300, 400, 2), _Taps(taps / taps.sum()))


def test_firtc_mixed_row_and_column_stages(cat):
    """Different row and column kernels (separate band tables and edge terms)."""
    _run(_frame(400, 520, 4), cat["g4_k16"], col_stage=cat["g16_k64"])
    _run(_frame(400, 520, 5), cat["sg38.4"], col_stage=cat["g2_k8"])


def test_firtc_kernel_nearly_as_long_as_the_line(cat):
    """385 taps on 388-sample lines: every output reaches both extensions."""
    _run(_frame(392, 388, 6), cat["sg38.4"])


def test_firtc_dense_detections_and_lap_scale(cat):
    """frac = 0.05 on white noise (thousands of detections through the
    per-CTA buffers, the global list and the finaliser's large-list path),
    with a sigma^2 scale on L."""
    x = np.random.default_rng(7).standard_normal((1024, 1024)).astype(np.float32)
    el, n_gpu, n_ref = _run(x, cat["g2_k8"], frac=0.05, lap_scale=4.0)
    assert n_ref > 4096


def test_firtc_default_dispatch(cat, monkeypatch):
    """Without the override, long kernels take the tensor cores and short
    ones the fp64 path."""
    from paper_1912_07133_b200 import _lib, detect

    monkeypatch.delenv("VMF_FORCE_FIRTC")
    x = _frame(256, 256, 8)
    for name, tc in (("g2_k8", False), ("g4_k16", True), ("g16_k64", True)):
        _lib.profile_begin()
        detect.blur_laplacian_detect(x, cat[name])
        torch.cuda.synchronize()
        _lib.profile_stop()
        assert ("firtc_rows" in _lib.profile_read()) == tc, name
