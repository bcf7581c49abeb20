"""Image files: PGM (P2/P5, 8/16-bit) and the raw float32 grid format
(pgmio.py of the reference).

read_pgm / write_pgm / read_f32 / write_f32 keep the reference's signatures
and results (PGM samples as float64 in [0, 1], i.e. divided by maxval; the
f32 format is a little-endian uint32 width, height header and row-major
float32 samples).

For the GPU stream the conversion is not done on the host: read_pgm_raw
returns the file's sample bytes untouched (big-endian u16 for maxval > 255,
else u8), read with one readinto() straight into a caller buffer (a pinned
staging tensor), and the row pass converts them (dtype codes VMF_U16BE /
VMF_U8: the byte swap is one PRMT per sample in the load).  The blur is
linear, so passing lap_scale = 1 / maxval reproduces the reference's units.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

__all__ = ["read_pgm", "write_pgm", "read_f32", "write_f32", "PgmInfo", "pgm_info",
           "read_pgm_raw"]


@dataclass(frozen=True)
class PgmInfo:
    width: int
    height: int
    maxval: int
    offset: int      # byte offset of the first sample
    binary: bool     # P5 (raw) or P2 (ASCII)

    @property
    def sample_dtype(self) -> np.dtype:
        return np.dtype(">u2") if self.maxval > 255 else np.dtype("u1")

    @property
    def nbytes(self) -> int:
        return self.width * self.height * self.sample_dtype.itemsize


def _parse_header(head: bytes, path: str) -> PgmInfo:
    if head[:2] not in (b"P2", b"P5"):
        raise ValueError(f"{path}: not a PGM file (P2/P5)")
    pos, tokens = 2, []
    while len(tokens) < 3:  # width, height, maxval; '#' comments run to end of line
        while pos < len(head) and head[pos:pos + 1].isspace():
            pos += 1
        if head[pos:pos + 1] == b"#":
            while pos < len(head) and head[pos:pos + 1] not in (b"\n", b"\r"):
                pos += 1
            continue
        start = pos
        while pos < len(head) and not head[pos:pos + 1].isspace():
            pos += 1
        if start == pos:
            raise ValueError(f"{path}: truncated PGM header")
        tokens.append(head[start:pos])
    try:
        width, height, maxval = (int(t) for t in tokens)
    except ValueError:
        raise ValueError(f"{path}: bad PGM dimensions/maxval") from None
    if width < 1 or height < 1 or not 0 < maxval < 65536:
        raise ValueError(f"{path}: bad PGM dimensions/maxval")
    binary = head[:2] == b"P5"
    return PgmInfo(width, height, maxval, pos + 1 if binary else pos, binary)


def pgm_info(path: str) -> PgmInfo:
    """Header of a PGM file (the header is read, the samples are not)."""
    with open(path, "rb") as fh:
        head = fh.read(1 << 16)
    return _parse_header(head, path)


def read_pgm(path: str) -> np.ndarray:
    """float64 [h, w] in [0, 1] (samples / maxval), as pgmio.py:15-53."""
    with open(path, "rb") as fh:
        data = fh.read()
    info = _parse_header(data, path)
    n = info.width * info.height
    if info.binary:
        raw = np.frombuffer(data, dtype=info.sample_dtype, count=min(n, (len(data) - info.offset)
                                                                     // info.sample_dtype.itemsize),
                            offset=min(info.offset, len(data)))
        if raw.size != n:
            raise ValueError(f"{path}: truncated PGM pixel data")
        img = raw.astype(np.float64).reshape(info.height, info.width)
    else:
        vals = np.array(data[info.offset:].split(), dtype=np.float64)
        if vals.size != n:
            raise ValueError(f"{path}: expected {n} samples")
        img = vals.reshape(info.height, info.width)
    return img / info.maxval


def read_pgm_raw(path: str, out=None):
    """(samples, info): the P5 sample bytes as a [h, w] array of the file's
    own type ('>u2' or 'u1'), no conversion.  `out` (any writable buffer of
    at least info.nbytes bytes, e.g. a pinned torch.uint8 tensor's numpy
    view) receives the bytes with one readinto(); the returned array views
    it."""
    with open(path, "rb") as fh:
        info = _parse_header(fh.read(1 << 16), path)
        if not info.binary:
            raise ValueError(f"{path}: read_pgm_raw needs a binary (P5) PGM")
        fh.seek(info.offset)
        if out is None:
            out = np.empty(info.nbytes, dtype=np.uint8)
        mv = memoryview(out).cast("B")
        if mv.nbytes < info.nbytes:
            raise ValueError(f"buffer of {mv.nbytes} bytes < {info.nbytes}")
        got = fh.readinto(mv[:info.nbytes])
        if got != info.nbytes:
            raise ValueError(f"{path}: truncated PGM pixel data")
    arr = np.frombuffer(mv[:info.nbytes], dtype=info.sample_dtype).reshape(info.height,
                                                                           info.width)
    return arr, info


def write_pgm(path: str, img, maxval: int = 255, binary: bool = True) -> None:
    """Clip to [0, 1], quantise to maxval levels (round half to even),
    write P5 (big-endian for maxval > 255) or P2 (pgmio.py:56-70)."""
    if not 0 < maxval < 65536:
        raise ValueError("maxval must be in 1..65535")
    a = np.clip(np.asarray(img, dtype=np.float64), 0.0, 1.0)
    q = np.rint(a * maxval).astype(np.uint16 if maxval > 255 else np.uint8)
    h, w = q.shape
    with open(path, "wb") as fh:
        fh.write(f"{'P5' if binary else 'P2'}\n{w} {h}\n{maxval}\n".encode("ascii"))
        if binary:
            fh.write(q.astype(">u2" if maxval > 255 else "u1").tobytes())
        else:
            fh.write(b"".join((" ".join(map(str, row.tolist())) + "\n").encode("ascii")
                              for row in q))


def read_f32(path: str) -> np.ndarray:
    """float64 [h, w] from the raw float32 format (pgmio.py:73-82)."""
    with open(path, "rb") as fh:
        head = fh.read(8)
        if len(head) != 8:
            raise ValueError(f"{path}: truncated float32 header")
        w, h = struct.unpack("<II", head)
        data = np.frombuffer(fh.read(), dtype="<f4")
    if data.size < w * h:
        raise ValueError(f"{path}: truncated float32 pixel data")
    return data[:w * h].astype(np.float64).reshape(h, w)


def write_f32(path: str, img) -> None:
    a = np.asarray(img, dtype=np.float64)
    h, w = a.shape
    with open(path, "wb") as fh:
        fh.write(struct.pack("<II", w, h))
        fh.write(a.astype("<f4").tobytes())
