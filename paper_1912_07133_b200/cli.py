"""Command-line front end routed to the GPU (cli.py of the reference,
SURVEY.md §8(f)4).

    python -m paper_1912_07133_b200.cli design --family repeated_pole --sigma 4 --out f.json
    python -m paper_1912_07133_b200.cli apply  --in img.pgm --coeff f.json --out out.f32
    python -m paper_1912_07133_b200.cli detect --in img.pgm --lambda 16
    python -m paper_1912_07133_b200.cli scene  --out scene.pgm

Same subcommand names, options, coefficient JSON schemas (polyz.py:575-630)
and exit codes (0 success, 2 usage or validation error, 3 numerical
failure) as the reference (cli.py:176-262).  `apply` and `detect` run on the
B200 kernels; `--threads` is accepted for compatibility and ignored (the
work is on the GPU).  `respond` and `bench` (frequency-response CSVs, the
reference's CPU timing harness) are outside the hot path and not provided.
"""
from __future__ import annotations

import argparse
import json
import math
import sys

import numpy as np

from . import design as D
from .errors import FilterError
from .filters import FirKernel, ThreePartIIR, gaussian_fir
from .pgmio import read_f32, read_pgm, write_f32, write_pgm

FAMILIES = ("interp_diff", "gaussian_fir", "fir_vm_bank", "colored_sg", "repeated_pole",
            "butterworth", "blunt_exponential", "butterworth_appendix")  # design.py:103-112


# ---------------------------------------------------------------------------
# coefficient JSON (the reference's two schemas)
# ---------------------------------------------------------------------------
def fir_to_json(k: FirKernel) -> dict:
    """{"k", "num", "den"}: num holds the z^-K..z^K coefficients c_m with
    taps(m) = c_-m; den is the unit polynomial (polyz.py:575-583)."""
    kk = k.k
    return {"k": kk, "num": [float(t) for t in reversed(k.taps)],
            "den": [0.0] * kk + [1.0] + [0.0] * kk}


def iir_to_json(f: ThreePartIIR) -> dict:
    return {"b_plus": list(f.b_plus), "a_plus": list(f.a_plus), "b_zero": f.b_zero,
            "parity": f.parity}


def stage_from_json(obj: dict):
    """ThreePartIIR or FirKernel from either schema (load_filter,
    polyz.py:625-633, and cli.py:44-63)."""
    if "b_plus" in obj:
        return ThreePartIIR(tuple(obj["b_plus"]), tuple(obj["a_plus"]), float(obj["b_zero"]),
                            obj["parity"])
    if "num" in obj and "den" in obj:
        k = int(obj["k"])
        num, den = [float(v) for v in obj["num"]], [float(v) for v in obj["den"]]
        if len(num) != 2 * k + 1 or len(den) != 2 * k + 1:
            raise ValueError("coefficient arrays must have length 2K+1")
        # strip zero padding, then require a pure FIR (den = unit at the centre)
        while k > 0 and num[0] == 0.0 and num[-1] == 0.0 and den[0] == 0.0 and den[-1] == 0.0:
            num, den, k = num[1:-1], den[1:-1], k - 1
        if any(v != 0.0 for i, v in enumerate(den) if i != k) or den[k] == 0.0:
            raise ValueError("filter is not FIR")
        taps = tuple(v / den[k] for v in reversed(num))
        if all(abs(taps[k - m] + taps[k + m]) <= 1e-12 * max(map(abs, taps)) for m in
               range(1, k + 1)) and taps[k] == 0.0 and k > 0:
            return FirKernel(taps, "anti", 1)
        return FirKernel(taps, "sym", 0 if abs(sum(taps) - 1.0) <= 1e-9 else 2)
    raise ValueError("unrecognized coefficient JSON (expected num/den or b_plus/a_plus)")


def load_stage(path: str):
    with open(path) as fh:
        return stage_from_json(json.load(fh))


def save_stage(path: str, f) -> None:
    obj = iir_to_json(f) if isinstance(f, ThreePartIIR) else fir_to_json(f)
    with open(path, "w") as fh:
        json.dump(obj, fh, indent=1)
        fh.write("\n")


def build(family: str, sigma: float = 0.0, d: int = 0, Dm: int = 3, l_pi_bar: int = 2,
          k=None, cascade_mode: str = "behind_blur"):
    """DesignSpec + build (design.py:92-149) over the re-implemented designs."""
    if family not in FAMILIES:
        raise ValueError(f"unknown family '{family}'")
    if Dm % 2 != 1 or Dm < 1:
        raise ValueError("D must be odd and >= 1")
    if l_pi_bar < 0:
        raise ValueError("l_pi_bar must be >= 0")
    if family not in ("interp_diff", "fir_vm_bank") and sigma <= 0:
        raise ValueError("sigma must be positive")
    l_d = (Dm - 1) // 2
    if family == "interp_diff":
        return D.interp_diff(d)
    if family == "gaussian_fir":
        return gaussian_fir(sigma, d, k if k is not None else math.ceil(5 * sigma))
    if family == "fir_vm_bank":
        return D.fir_vm_bank(Dm, l_pi_bar, cascade_mode)
    if family == "repeated_pole":
        return D.repeated_pole_blur(sigma, l_d, l_pi_bar)
    if family == "butterworth":
        return D.butterworth_blur(sigma, l_d)
    if family == "blunt_exponential":
        return D.blunt_exponential_blur(sigma, k or 3)
    if family == "butterworth_appendix":
        return D.butterworth_appendix(sigma)
    return D.colored_sg_blur(sigma, l_d)


# ---------------------------------------------------------------------------
# subcommands
# ---------------------------------------------------------------------------
def _read_image(path: str) -> np.ndarray:
    return read_f32(path) if path.endswith(".f32") else read_pgm(path)


def _write_image(path: str, img) -> None:
    (write_f32 if path.endswith(".f32") else write_pgm)(path, img)


def _cmd_design(args) -> int:
    f = build(args.family, args.sigma, args.d, args.D, args.l_pi_bar, args.k, args.cascade_mode)
    if isinstance(f, list):
        with open(args.out, "w") as fh:
            json.dump({"bank": [fir_to_json(k) for k in f]}, fh, indent=1)
            fh.write("\n")
        for i, k in enumerate(f):
            print(f"kernel d={i}: {len(k.taps)} taps, parity {k.parity}")
    else:
        save_stage(args.out, f)
        if isinstance(f, ThreePartIIR):
            print(f"three-part IIR, K={f.k}, b_zero={f.b_zero:.12g}")
        else:
            print(f"FIR, {len(f.taps)} taps, parity {f.parity}, d={f.d}")
    return 0


def _cmd_apply(args) -> int:
    from . import engine

    img = _read_image(args.input)
    stage = load_stage(args.coeff)
    if args.axis in ("x", "both"):
        img = engine.apply_rows(img, stage)
    if args.axis in ("y", "both"):
        img = engine.apply_cols(img, stage)
    img = np.asarray(img, dtype=np.float64)
    if args.crop_border:
        n = args.crop_border
        if 2 * n >= min(img.shape):
            raise ValueError("crop larger than image")
        img = img[n:-n, n:-n]
    _write_image(args.out, img)
    return 0


def _cmd_detect(args) -> int:
    from . import blob

    img = _read_image(args.input)
    t1 = args.t1
    if t1 is None:
        t1 = blob.calibrate_t1(args.lam, args.family, args.ecc, args.polarity)
    dets = blob.detect(img, args.lam, args.family, t1, args.t2, args.polarity)
    for det in dets:
        print(det.to_json())
    print(f"{len(dets)} detections (t1={t1:.6g})", file=sys.stderr)
    if args.overlay:
        out = np.array(img, dtype=np.float64, copy=True)  # blob.py:208-214
        hi = max(1.0, float(out.max()))
        for det in dets:
            out[det.y, det.x] = hi
        _write_image(args.overlay, out)
    return 0


def _cmd_scene(args) -> int:
    from .blob import ellipse_grid_scene, render_scene, scene_from_json

    if args.spec:
        with open(args.spec) as fh:
            scene = scene_from_json(json.load(fh))
    else:
        scene = ellipse_grid_scene({"ecc2": 2.0, "ecc4": 4.0}[args.preset])
    _write_image(args.out, render_scene(scene, args.supersample))
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="vmfilt-b200", description=__doc__,
                                 formatter_class=argparse.RawDescriptionHelpFormatter)
    sub = ap.add_subparsers(dest="command", required=True)

    p = sub.add_parser("design", help="build a filter and save coefficients")
    p.add_argument("--family", required=True, choices=FAMILIES)
    p.add_argument("--sigma", type=float, default=0.0)
    p.add_argument("--d", type=int, default=0)
    p.add_argument("--D", type=int, default=3)
    p.add_argument("--l-pi-bar", type=int, default=2)
    p.add_argument("--k", type=int, default=None)
    p.add_argument("--cascade-mode", default="behind_blur", choices=("behind_blur", "standalone"))
    p.add_argument("--order", type=int, default=None, help="accepted for compatibility")
    p.add_argument("--out", required=True)
    p.set_defaults(func=_cmd_design)

    p = sub.add_parser("apply", help="filter an image with saved coefficients (GPU)")
    p.add_argument("--in", dest="input", required=True)
    p.add_argument("--coeff", required=True)
    p.add_argument("--out", required=True)
    p.add_argument("--axis", default="both", choices=("x", "y", "both"))
    p.add_argument("--crop-border", type=int, default=0)
    p.add_argument("--threads", default="max", help="ignored (GPU)")
    p.set_defaults(func=_cmd_apply)

    p = sub.add_parser("detect", help="scale-selective blob detection (GPU)")
    p.add_argument("--in", dest="input", required=True)
    p.add_argument("--lambda", dest="lam", type=float, required=True)
    p.add_argument("--family", default="gaussian_fir")
    p.add_argument("--t1", type=float, default=None)
    p.add_argument("--t2", type=float, default=None)
    p.add_argument("--ecc", type=float, default=2.0)
    p.add_argument("--polarity", default="dark", choices=("dark", "bright"))
    p.add_argument("--overlay", default=None)
    p.add_argument("--threads", default="max", help="ignored (GPU)")
    p.set_defaults(func=_cmd_detect)

    p = sub.add_parser("scene", help="render a synthetic ellipse image")
    p.add_argument("--out", required=True)
    p.add_argument("--preset", default="ecc2", choices=("ecc2", "ecc4"))
    p.add_argument("--spec", default=None)
    p.add_argument("--supersample", type=int, default=4)
    p.set_defaults(func=_cmd_scene)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except FilterError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 3
    except (ValueError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
