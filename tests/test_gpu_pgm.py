"""The integer sample types of the first pass (u8, big-endian u16) and the
PGM stream front end: conversions inside the row pass are
exact, so every path is bit-identical to the fp32 path on the same values,
and the PGM stream reproduces the reference's units (read_pgm / maxval)."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1912_07133_b200 import pgmio, synth
from tests.parity import TOL_REL, compare_blobs, max_rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"


def _E():
    from paper_1912_07133_b200 import engine

    return engine


def _D():
    from paper_1912_07133_b200 import detect

    return detect


@pytest.mark.parametrize("name", ["rp4", "bw6", "sg3.2", "g4_k16"])
@pytest.mark.parametrize("shape", [(96, 4096), (67, 131)])
def test_integer_samples(cat, name, shape):
    """Big-endian u16 and u8 go through the same kernels as host-order u16:
    bit-identical results.  Against the fp32 input path (a different row-pass
    variant for widths that are multiples of 32) within a few fp32 ulps."""
    E = _E()
    rng = np.random.default_rng(7)
    v16 = rng.integers(0, 65536, size=shape).astype(np.uint16)
    v8 = rng.integers(0, 256, size=shape).astype(np.uint8)
    st = cat[name]
    native = E.apply_rows(v16, st)
    np.testing.assert_array_equal(E.apply_rows(v16.astype(">u2"), st), native)
    np.testing.assert_array_equal(E.apply_rows(v8, st), E.apply_rows(v8.astype(np.uint16), st))
    ref = E.apply_rows(v16.astype(np.float32), st)
    assert np.abs(native - ref).max() <= 4e-6 * np.abs(ref).max()


@pytest.mark.parametrize("name", ["rp6", "sg3.2"])
def test_fused_detect_big_endian(cat, name):
    D = _D()
    x = synth.config4_stream(n_frames=1, size=512)[0]
    a = D.blur_laplacian_detect(x, cat[name], frac=0.5, lap_scale=1 / 4095)
    b = D.blur_laplacian_detect(x.astype(">u2"), cat[name], frac=0.5, lap_scale=1 / 4095)
    assert a.count == b.count
    np.testing.assert_array_equal(a.y, b.y)
    np.testing.assert_array_equal(a.x, b.x)
    np.testing.assert_array_equal(a.value, b.value)


@pytest.mark.parametrize("maxval", [4095, 255])
def test_pgm_stream_matches_reference_units(tmp_path, cat, maxval):
    """Frames written as PGM (16-bit big-endian or 8-bit), streamed from disk:
    each frame equals the single call on the same samples, and the L values
    are in the reference's units (read_pgm's [0, 1] image)."""
    D = _D()
    frames = synth.config4_stream(n_frames=3, size=512)
    paths = []
    for i, f in enumerate(frames):
        p = str(tmp_path / f"f{i}.pgm")
        pgmio.write_pgm(p, f.astype(np.float64) / 4095.0, maxval=maxval)
        paths.append(p)
    got = D.pgm_stream_detect(paths, cat["rp6"], frac=0.5)
    assert len(got) == 3
    for p, g in zip(paths, got):
        raw, info = pgmio.read_pgm_raw(p)
        one = D.blur_laplacian_detect(raw, cat["rp6"], frac=0.5, lap_scale=1.0 / info.maxval)
        assert g.count == one.count
        np.testing.assert_array_equal(g.y, one.y)
        np.testing.assert_array_equal(g.x, one.x)
        np.testing.assert_array_equal(g.value, one.value)
    # the first frame against the oracle on the reference's reader output
    img = pgmio.read_pgm(paths[0])
    B, L, (ys, xs, vs, thr) = O.pipeline(img, cat["rp6"], frac=0.5)
    dets, blur, lap = D.blur_laplacian_detect(pgmio.read_pgm_raw(paths[0])[0], cat["rp6"],
                                              frac=0.5, lap_scale=1.0 / maxval,
                                              return_fields=True)
    assert max_rel_err(lap, L) < TOL_REL
    exempt, bad = compare_blobs(dets.as_set(), set(zip(ys.tolist(), xs.tolist())), L, thr)
    assert not bad, bad[:10]


def test_pgm_stream_rejects_mixed_frames(tmp_path, cat):
    D = _D()
    a, b = str(tmp_path / "a.pgm"), str(tmp_path / "b.pgm")
    pgmio.write_pgm(a, np.zeros((64, 64)), maxval=4095)
    pgmio.write_pgm(b, np.zeros((64, 32)), maxval=4095)
    with pytest.raises(ValueError):
        D.pgm_stream_detect([a, b], cat["rp6"])
