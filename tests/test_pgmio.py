"""PGM / raw-f32 file I/O (pgmio.py of the reference): byte-exact writer,
reader semantics (samples / maxval, '#' comments, P2 and P5, 8/16-bit),
the zero-conversion raw reader used by the GPU stream, and the errors."""
import os

import numpy as np
import pytest

from paper_1912_07133_b200 import pgmio as P


@pytest.mark.parametrize("maxval", [7, 255, 4095, 65535])
@pytest.mark.parametrize("binary", [True, False])
def test_round_trip(tmp_path, maxval, binary):
    img = np.random.default_rng(maxval).random((13, 17))
    f = str(tmp_path / "a.pgm")
    P.write_pgm(f, img, maxval, binary)
    q = np.rint(np.clip(img, 0, 1) * maxval)
    assert np.array_equal(P.read_pgm(f), q / maxval)
    head = open(f, "rb").read(20)
    assert head.startswith(b"P5\n17 13\n" if binary else b"P2\n17 13\n")
    if binary:
        raw, info = P.read_pgm_raw(f)
        assert (info.width, info.height, info.maxval) == (17, 13, maxval)
        assert raw.dtype == (np.dtype(">u2") if maxval > 255 else np.dtype("u1"))
        assert np.array_equal(raw.astype(np.float64), q)
        # big-endian on disk: the first sample's high byte comes first
        body = open(f, "rb").read()[info.offset:]
        if maxval > 255:
            assert body[0] * 256 + body[1] == q[0, 0]


def test_header_comments_and_raw_into_buffer(tmp_path):
    f = str(tmp_path / "c.pgm")
    with open(f, "wb") as fh:
        fh.write(b"P5\n# made by hand\n3 2 # trailing\n255\n" + bytes(range(10, 16)))
    assert np.array_equal(P.read_pgm(f) * 255, [[10, 11, 12], [13, 14, 15]])
    buf = np.zeros(64, dtype=np.uint8)
    raw, info = P.read_pgm_raw(f, out=buf)
    assert info.nbytes == 6 and list(buf[:6]) == list(range(10, 16))
    assert np.shares_memory(raw, buf)
    with pytest.raises(ValueError):
        P.read_pgm_raw(f, out=np.zeros(4, dtype=np.uint8))


def test_errors(tmp_path):
    f = str(tmp_path / "bad.pgm")
    for content in (b"P6\n2 2\n255\n" + bytes(12), b"P5\n2 2\n", b"P5\n0 2\n255\n",
                    b"P5\n2 2\n70000\n" + bytes(8), b"P5\n2 2\n255\n" + bytes(3),
                    b"P2\n2 2\n255\n1 2 3\n"):
        with open(f, "wb") as fh:
            fh.write(content)
        with pytest.raises(ValueError):
            P.read_pgm(f)
    with pytest.raises(ValueError):
        P.write_pgm(f, np.zeros((2, 2)), maxval=0)
    g = str(tmp_path / "t.f32")
    with open(g, "wb") as fh:
        fh.write(b"\x02\x00\x00\x00\x02\x00\x00\x00" + bytes(8))
    with pytest.raises(ValueError):
        P.read_f32(g)


def test_f32_round_trip(tmp_path):
    img = np.random.default_rng(1).standard_normal((5, 9))
    f = str(tmp_path / "x.f32")
    P.write_f32(f, img)
    assert os.path.getsize(f) == 8 + 4 * 45
    assert np.array_equal(P.read_f32(f), img.astype(np.float32).astype(np.float64))
