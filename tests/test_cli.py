"""Command-line front end (cli.py of the reference): design writes the
reference's coefficient schemas, scene renders, exit codes 0/2/3; apply and
detect run on the GPU and agree with the Python API."""
import json

import numpy as np
import pytest

from paper_1912_07133_b200 import cli, design, filters, pgmio


def test_design_schemas_round_trip(tmp_path):
    out = str(tmp_path / "f.json")
    assert cli.main(["design", "--family", "repeated_pole", "--sigma", "4", "--out", out]) == 0
    f = cli.load_stage(out)
    assert f == design.repeated_pole_blur(4.0)
    assert cli.main(["design", "--family", "gaussian_fir", "--sigma", "2", "--out", out]) == 0
    obj = json.load(open(out))
    assert obj["k"] == 10 and obj["den"][10] == 1.0 and len(obj["num"]) == 21
    assert cli.load_stage(out) == filters.gaussian_fir(2.0, 0, 10)
    assert cli.main(["design", "--family", "interp_diff", "--d", "1", "--out", out]) == 0
    k = cli.load_stage(out)
    assert (k.taps, k.parity, k.d) == ((0.5, 0.0, -0.5), "anti", 1)
    assert cli.main(["design", "--family", "fir_vm_bank", "--out", out]) == 0
    assert len(json.load(open(out))["bank"]) == 3


def test_exit_codes(tmp_path, capsys):
    out = str(tmp_path / "f.json")
    assert cli.main(["design", "--family", "repeated_pole", "--sigma", "64", "--out", out]) == 3
    assert cli.main(["design", "--family", "repeated_pole", "--sigma", "0.5", "--out", out]) == 2
    assert cli.main(["design", "--family", "colored_sg", "--sigma", "0.5", "--out", out]) == 2
    assert cli.main(["apply", "--in", str(tmp_path / "missing.pgm"), "--coeff", out, "--out",
                     out]) == 2
    with pytest.raises(SystemExit):
        cli.main(["design", "--family", "nope", "--out", out])
    with open(out, "w") as fh:
        json.dump({"k": 1, "num": [0, 1, 0], "den": [0.5, 1, 0.5]}, fh)
    with pytest.raises(ValueError):
        cli.load_stage(out)


def test_scene(tmp_path):
    out = str(tmp_path / "s.pgm")
    assert cli.main(["scene", "--out", out, "--supersample", "2"]) == 0
    img = pgmio.read_pgm(out)
    assert img.shape == (768, 1024) and img.min() == 0.0 and img.max() == 1.0


@pytest.mark.gpu
def test_apply_and_detect_on_gpu(tmp_path, capsys):
    from paper_1912_07133_b200 import blob, engine

    scene = str(tmp_path / "s.pgm")
    assert cli.main(["scene", "--out", scene]) == 0
    coeff = str(tmp_path / "f.json")
    assert cli.main(["design", "--family", "repeated_pole", "--sigma", "4", "--out", coeff]) == 0
    out = str(tmp_path / "o.f32")
    assert cli.main(["apply", "--in", scene, "--coeff", coeff, "--out", out,
                     "--crop-border", "3"]) == 0
    img = pgmio.read_pgm(scene)
    f = design.repeated_pole_blur(4.0)
    want = engine.apply_cols(engine.apply_rows(img, f), f)[3:-3, 3:-3]
    np.testing.assert_array_equal(pgmio.read_f32(out), np.asarray(want, np.float32))
    capsys.readouterr()
    assert cli.main(["detect", "--in", scene, "--lambda", "16", "--t1", "0.01"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    dets = blob.detect(img, 16.0, "gaussian_fir", 0.01)
    assert [json.loads(s) for s in lines] == [json.loads(d.to_json()) for d in dets]
    assert len(dets) > 0
