"""Hessian blob detector: the scene renderer and the
oracle restatement of blob.detect, pinned to the reference's own outputs
(tests/golden/blob_golden.json, made by tests/golden/make_blob_golden.py).
CPU only; the GPU detector is checked in tests/test_gpu_blob.py."""
import hashlib
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1912_07133_b200 import blob as B
from paper_1912_07133_b200.filters import gaussian_fir

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(HERE, "golden", "blob_golden.json")) as fh:
        return json.load(fh)


def _digest(img):
    return hashlib.sha256(np.ascontiguousarray(img, dtype=np.float64).tobytes()).hexdigest()


def _twins():
    return B.render_scene(B.EllipseScene(96, 80, (B.Ellipse(30, 40, 8.0), B.Ellipse(60, 40, 8.0))))


def test_render_scene_bit_identical(gold):
    assert _digest(B.render_scene(B.ellipse_grid_scene(2.0))) == gold["ecc2"]["digest"]["sha256"]
    assert _digest(B.render_scene(B.ellipse_grid_scene(4.0))) == gold["ecc4"]["digest"]["sha256"]
    assert _digest(_twins()) == gold["twins"]["digest"]["sha256"]


def test_render_scene_area_and_bounds():
    img = B.render_scene(B.EllipseScene(101, 101, (B.Ellipse(50, 50, 20, 1.0, 0.0),)))
    assert float((1.0 - img).sum()) == pytest.approx(math.pi * 400, rel=2e-3)
    with pytest.raises(ValueError):
        B.render_scene(B.EllipseScene(64, 64, (B.Ellipse(2, 2, 10, 1.0, 0.0),)))


def test_scene_json_round_trip():
    obj = {"width": 64, "height": 48, "background": 0.9,
           "ellipses": [{"cx": 30, "cy": 20, "a": 5, "ecc": 2.0, "theta": 0.3}]}
    sc = B.scene_from_json(json.loads(json.dumps(obj)))
    assert (sc.width, sc.height, sc.ellipses[0].a, sc.background) == (64, 48, 5.0, 0.9)


def _close_dets(got, ref, nd_rel=1e-9):
    assert [(g[0], g[1]) for g in got] == [(r[0], r[1]) for r in ref]
    for g, r in zip(got, ref):
        assert g[4] == pytest.approx(r[4], rel=nd_rel)
        for a, b in ((g[2], r[2]), (g[3], r[3])):
            assert (math.isnan(a) and math.isnan(b)) or a == pytest.approx(b, rel=1e-7, abs=1e-9)


def test_oracle_detect_matches_reference(gold):
    img = B.render_scene(B.ellipse_grid_scene(2.0))
    g = gaussian_fir(8.0, 0, 40)
    _close_dets(O.hessian_detect(img, g, 16.0, gold["ecc2"]["t1"]), gold["ecc2"]["dark"])
    _close_dets(O.hessian_detect(1.0 - img, g, 16.0, gold["ecc2"]["t1"], polarity="bright"),
                gold["ecc2"]["bright"])
    tw = _twins()
    got = O.hessian_detect(tw, gaussian_fir(4.0, 0, 20), 8.0, gold["twins"]["t1"])
    _close_dets(got, gold["twins"]["dets"])
    assert [(d[0], d[1]) for d in got] == [(30, 40), (60, 40)] and got[0][4] == got[1][4]


def test_oracle_t2_sweep_matches_reference(gold):
    img = B.render_scene(B.ellipse_grid_scene(4.0))
    g = gaussian_fir(8.0, 0, 40)
    for t2, ref in gold["ecc4"]["t2"].items():
        _close_dets(O.hessian_detect(img, g, 16.0, gold["ecc4"]["t1"], t2=float(t2)), ref)


def test_oracle_calibration_peak_matches_reference(gold):
    # calibrate_t1 = factor * max nd over the polarity mask of one matched ellipse
    a = 8.0
    pad = int(math.ceil(6 * a))
    img = B.render_scene(B.EllipseScene(2 * pad + 1, 2 * pad + 1, (B.Ellipse(pad, pad, a, 2.0),)))
    nd, tr, _, _ = O.hessian_fields(O.derivative_field(img, gaussian_fir(4.0, 0, 20)), 4.0)
    t1 = 0.7 * float(nd[tr > 0].max())
    assert t1 == pytest.approx(gold["t1_loose"]["t1"], rel=1e-12)
    assert gold["t1_loose"]["t1_half"] == pytest.approx(t1 * 5 / 7, rel=1e-9)


def test_detector_validation_mirrors_reference():
    img = np.ones((32, 32))
    with pytest.raises(ValueError):
        B.detect(img, 8.0, "gaussian_fir", 0.0)
    with pytest.raises(ValueError):
        B.detect(img, 8.0, "gaussian_fir", 1.0, polarity="grey")
    with pytest.raises(ValueError):
        B.detect(img, 8.0, "lanczos", 1.0)
