"""Golden outputs of the reference's Hessian blob detector (blob.py), used by
tests/test_blob.py to pin the oracle restatement (oracle.hessian_detect), the
scene renderer and the GPU detector.

Run HERE, where /root/reference exists:   python tests/golden/make_blob_golden.py
It imports the reference package from a scratch copy (NUMBA_CACHE_DIR
redirected; nothing is written into /root/reference) and records, for the
reference's own detector test scenes (tests/test_blob.py of the reference):
calibrate_t1 values, detect() results (x, y, dx, dy, ndet) and a digest of
each rendered scene.  Output: tests/golden/blob_golden.json.
"""
import hashlib
import json
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SCRATCH = "/tmp/vmf_refpkg"


def main():
    if not os.path.isdir(SCRATCH):
        shutil.copytree("/root/reference/pkg", SCRATCH)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/vmf_numba_cache")
    sys.path.insert(0, os.path.join(SCRATCH, "src"))
    import numpy as np
    from vmfilt.blob import (Ellipse, EllipseScene, calibrate_t1, detect, ellipse_grid_scene,
                             render_scene)

    def digest(img):
        a = np.ascontiguousarray(img, dtype=np.float64)
        return {"sha256": hashlib.sha256(a.tobytes()).hexdigest(), "sum": float(a.sum()),
                "shape": list(a.shape)}

    def dets(ds):
        return [[d.x, d.y, d.dx, d.dy, d.ndet] for d in ds]

    out = {}
    ecc2 = render_scene(ellipse_grid_scene(2.0))
    ecc4 = render_scene(ellipse_grid_scene(4.0))
    t1_2 = calibrate_t1(16.0, "gaussian_fir", 2.0)
    t1_4 = calibrate_t1(16.0, "gaussian_fir", 4.0)
    out["ecc2"] = {"digest": digest(ecc2), "t1": t1_2,
                   "dark": dets(detect(ecc2, 16.0, "gaussian_fir", t1_2)),
                   "bright": dets(detect(1.0 - ecc2, 16.0, "gaussian_fir", t1_2,
                                         polarity="bright"))}
    out["ecc4"] = {"digest": digest(ecc4), "t1": t1_4,
                   "t2": {str(t2): dets(detect(ecc4, 16.0, "gaussian_fir", t1_4, t2=t2))
                          for t2 in (16.0, 8.0, 4.0, 2.0, 1.0)}}
    twins = render_scene(EllipseScene(96, 80, (Ellipse(30, 40, 8.0), Ellipse(60, 40, 8.0))))
    t1_t = calibrate_t1(8.0, "gaussian_fir", 1.0, factor=0.9)
    out["twins"] = {"digest": digest(twins), "t1": t1_t,
                    "dets": dets(detect(twins, 8.0, "gaussian_fir", t1_t))}
    out["t1_loose"] = {"t1": calibrate_t1(8.0, "gaussian_fir", 2.0),
                       "t1_half": calibrate_t1(8.0, "gaussian_fir", 2.0, factor=0.5)}
    with open(os.path.join(HERE, "blob_golden.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote", os.path.join(HERE, "blob_golden.json"),
          {k: len(v.get("dark", v.get("dets", []))) if isinstance(v, dict) else 0
           for k, v in out.items()})


if __name__ == "__main__":
    main()
