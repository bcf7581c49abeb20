"""Seeded synthetic frames for the five BASELINE.json configs.

The reference has no image dataset for this path (its paper's aerial images
are not shipped; SPEC.md:8 substitutes synthetic scenes), so every config is
generated here from SURVEY.md §8(d): isotropic Gaussian blobs
A * exp(-r^2 / 2 s^2) rendered over +-5 s, centres uniform over the whole
frame, added to Gaussian noise; numpy.random.default_rng(seed) with a fixed
seed per config; generated in float64 and cast to the config dtype once, so
the oracle and the GPU consume the same stored array.
"""
from __future__ import annotations

import math

import numpy as np

SEEDS = {1: 1, 2: 1, 3: 3, 4: 4, 5: 5}


def _add_blob(img, cy, cx, s, amp):
    h, w = img.shape
    r = int(math.ceil(5 * s))
    y0, y1 = max(int(math.floor(cy)) - r, 0), min(int(math.floor(cy)) + r + 2, h)
    x0, x1 = max(int(math.floor(cx)) - r, 0), min(int(math.floor(cx)) + r + 2, w)
    if y0 >= y1 or x0 >= x1:
        return
    gy = np.exp(-((np.arange(y0, y1) - cy) ** 2) / (2 * s * s))
    gx = np.exp(-((np.arange(x0, x1) - cx) ** 2) / (2 * s * s))
    img[y0:y1, x0:x1] += amp * np.outer(gy, gx)


def blob_frame(h, w, n_blobs, s_lo, s_hi, a_lo, a_hi, noise_mean, noise_std, seed,
               log_uniform=False):
    rng = np.random.default_rng(seed)
    img = noise_mean + noise_std * rng.standard_normal((h, w))
    cy = rng.uniform(0, h - 1, n_blobs)
    cx = rng.uniform(0, w - 1, n_blobs)
    if log_uniform:
        s = np.exp(rng.uniform(math.log(s_lo), math.log(s_hi), n_blobs))
    else:
        s = rng.uniform(s_lo, s_hi, n_blobs)
    amp = rng.uniform(a_lo, a_hi, n_blobs)
    for i in range(n_blobs):
        _add_blob(img, cy[i], cx[i], s[i], amp[i])
    return img


def config1_frame(size: int = 512) -> np.ndarray:
    """512^2 fp32, N(0.1, 0.02^2) + 20 blobs (s = 4, A = 1)."""
    return blob_frame(size, size, 20, 4.0, 4.0, 1.0, 1.0, 0.1, 0.02, SEEDS[1]).astype(np.float32)


config2_frame = config1_frame  # same generator (BASELINE.json configs[1])


def config3_frame(size: int = 4096) -> np.ndarray:
    """4096^2 fp32, N(0, 0.05^2) + 2000 blobs, s log-uniform [2,32],
    A uniform [0.5, 1.5]."""
    n = max(1, int(round(2000 * (size / 4096) ** 2)))
    return blob_frame(size, size, n, 2.0, 32.0, 0.5, 1.5, 0.0, 0.05, SEEDS[3],
                      log_uniform=True).astype(np.float32)


def config4_stream(n_frames: int = 64, size: int = 2048) -> np.ndarray:
    """n_frames x size^2 uint16 in [0, 4095]: background 400 + 30 N(0,1)
    (rounded), 500 blobs s ~ U[3,12], A ~ U[200,800], each drifting in a
    fixed direction at U[1,3] px/frame."""
    rng = np.random.default_rng(SEEDS[4])
    n = max(1, int(round(500 * (size / 2048) ** 2)))
    cy = rng.uniform(0, size - 1, n)
    cx = rng.uniform(0, size - 1, n)
    s = rng.uniform(3.0, 12.0, n)
    amp = rng.uniform(200.0, 800.0, n)
    ang = rng.uniform(0, 2 * math.pi, n)
    spd = rng.uniform(1.0, 3.0, n)
    out = np.empty((n_frames, size, size), dtype=np.uint16)
    for f in range(n_frames):
        img = 400.0 + 30.0 * rng.standard_normal((size, size))
        for i in range(n):
            _add_blob(img, cy[i] + f * spd[i] * math.sin(ang[i]),
                      cx[i] + f * spd[i] * math.cos(ang[i]), s[i], amp[i])
        out[f] = np.clip(np.rint(img), 0, 4095).astype(np.uint16)
    return out


def config5_frame(size: int = 8192) -> np.ndarray:
    """8192^2 fp32, N(0, 0.05^2) + 5000 blobs, s log-uniform [8, 64]."""
    n = max(1, int(round(5000 * (size / 8192) ** 2)))
    return blob_frame(size, size, n, 8.0, 64.0, 0.5, 1.5, 0.0, 0.05, SEEDS[5],
                      log_uniform=True).astype(np.float32)


# The per-config pipelines; catalog names in data/catalog.json.
CONFIG_STAGES = {
    1: ["rp4", "rp4_k2"],
    2: ["sg3.2", "g4_k16"],
    3: {"iir": ["rp2", "rp4", "rp8", "rp16", "rp32"],
        "fir": ["g2_k8", "g4_k16", "g8_k32", "g16_k64", "g32_k128"],
        "sigmas": [2.0, 4.0, 8.0, 16.0, 32.0]},
    4: ["rp6"],
    5: ["bw48", "sg38.4"],
}
