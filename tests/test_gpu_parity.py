"""GPU parity against the CPU oracle (pinned to the reference by
tests/test_oracle.py).  Every call goes through the C ABI
(libvmfilt_b200.so) via the drop-in engine / detect API."""
import zlib

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1912_07133_b200 import filters as F
from paper_1912_07133_b200 import synth
from tests.parity import TOL_REL, compare_blobs, max_rel_err

pytestmark = pytest.mark.gpu

# fp32 output of an fp64-state pass: error is a few fp32 ulps of the output
PASS_TOL = 4e-6


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1912_07133_b200 import _lib

    _lib.lib()


def _E():
    from paper_1912_07133_b200 import engine

    return engine


def _D():
    from paper_1912_07133_b200 import detect

    return detect


def _f32(x):
    """The GPU consumes fp32; the oracle consumes the same values in fp64."""
    return np.asarray(x, dtype=np.float32)


@pytest.mark.parametrize("op", ["iir_rows", "iir_cols", "conv_rows", "conv_cols"])
def test_single_pass_matches_oracle(golden, cat, op):
    E = _E()
    n = 0
    for key in [k for k in golden if k.startswith(op + "/")]:
        _, fname, iname = key.split("/")
        x = _f32(golden[f"in/{iname}"])
        got = getattr(E, op)(x, cat[fname])
        want = getattr(O, op)(x, cat[fname])
        assert got.dtype == np.float32 and got.shape == want.shape
        assert max_rel_err(got, want) < PASS_TOL, key
        n += 1
    assert n > 10


def test_u16_input_path(golden, cat):
    E = _E()
    x = golden["in/u16"].astype(np.uint16)
    for name in ("rp4", "bw6", "g1.5_k8"):
        for op in ("apply_rows", "apply_cols"):
            got = getattr(E, op)(x, cat[name])
            want = getattr(O, op)(x.astype(np.float64), cat[name])
            assert max_rel_err(got, want) < PASS_TOL, (name, op)


def test_torch_in_torch_out(cat):
    E = _E()
    x = torch.rand(64, 80, device="cuda")
    y = E.apply_rows(x, cat["rp4"])
    assert isinstance(y, torch.Tensor) and y.is_cuda and y.dtype == torch.float32
    want = O.iir_rows(x.cpu().numpy(), cat["rp4"])
    assert max_rel_err(y.cpu().numpy(), want) < PASS_TOL


def test_constant_image_invariance_everywhere(cat):
    # tests/test_engine.py:49-53 / test_acceptance.py:175-183
    E = _E()
    x = np.full((40, 61), 3.7, np.float32)
    for name in ("rp4", "rp32", "bw48", "blunt4", "bwapp6", "g4_k16", "sg3.2"):
        f = cat[name]
        if min(x.shape) < (len(f.taps) if F.is_fir(f) else 2 * f.k + 1):
            continue
        y = E.apply_cols(E.apply_rows(x, f), f)
        assert np.abs(y - 3.7).max() <= 2e-6 * 3.7, name


def test_impulse_response_and_long_lines(cat):
    E = _E()
    for n in (101, 4099):  # 4099: many chunks plus a folded tail
        x = np.zeros((3, n), np.float32)
        x[1, n // 2] = 1.0
        for name in ("rp2", "rp32", "bw48"):
            got = E.iir_rows(x, cat[name])
            want = O.iir_rows(x, cat[name])
            assert np.abs(got - want).max() < 1e-7 * max(1, np.abs(want).max()), (name, n)
            got = E.iir_cols(np.ascontiguousarray(x.T), cat[name])
            assert np.abs(got.T - want).max() < 1e-7 * max(1, np.abs(want).max()), (name, n)


def test_all_orders_and_lengths(cat):
    # K = 1..4 (and K=0), line lengths around the chunk size and 2K+1
    E = _E()
    rng = np.random.default_rng(3)
    fs = [F.ThreePartIIR((0.2,), (-0.6,), 0.2, "sym"), cat["rp4_k2"], cat["rp4"], cat["rp4_k4"],
          F.ThreePartIIR((), (), 1.0, "sym"), F.ThreePartIIR((0.1, -0.05), (-0.9, 0.2), 0.0, "anti")]
    for f in fs:
        for n in sorted({2 * f.k + 1, 63, 64, 65, 64 + f.k - 1, 127, 128, 129, 300}):
            if n < 2 * f.k + 1:
                continue
            x = rng.standard_normal((5, n)).astype(np.float32)
            assert max_rel_err(E.iir_rows(x, f), O.iir_rows(x, f)) < PASS_TOL, (f, n)
            xt = np.ascontiguousarray(x.T)
            try:
                got = E.iir_cols(xt, f)
            except ValueError as e:
                raise AssertionError((f, n, xt.shape, xt.strides, str(e)))
            assert max_rel_err(got, O.iir_cols(xt, f)) < PASS_TOL, (f, n)


def test_step_inputs_match_transposed_form_reference(cat):
    # tests/test_engine.py:69-116: the steady-state initialisation
    E = _E()
    f = cat["rp4"]
    for lo, hi in ((2.0, 5.0), (4.0, -1.0), (0.0, 1.0)):
        x = np.array([[lo] * 25 + [hi] * 25] * 2, np.float32)
        got = E.iir_rows(x, f)
        want = O.iir_rows(x, f)
        assert np.abs(got - want).max() < 1e-5


def test_errors_mirror_reference(cat):
    E = _E()
    from paper_1912_07133_b200.errors import StabilityError

    bad = F.ThreePartIIR((0.5,), (-1.5,), 0.2, "sym")
    with pytest.raises(StabilityError):
        E.iir_rows(np.zeros((4, 16), np.float32), bad)
    with pytest.raises(ValueError):
        E.iir_rows(np.zeros((2, 6), np.float32), cat["rp4"])
    with pytest.raises(ValueError):
        E.conv_rows(np.zeros((4, 10), np.float32), cat["g4_k16"])
    with pytest.raises(ValueError):
        E.apply_rows(np.zeros((4,), np.float32), cat["rp4"])
    with pytest.raises(TypeError):
        E.apply_rows(np.zeros((4, 16), np.float32), object())


def test_run_to_run_determinism(cat):
    E = _E()
    x = torch.randn(300, 500, device="cuda")
    a = E.apply_cols(E.apply_rows(x, cat["rp8"]), cat["rp8"])
    b = E.apply_cols(E.apply_rows(x, cat["rp8"]), cat["rp8"])
    assert torch.equal(a, b)


@pytest.mark.parametrize("name", ["rp4_k2", "rp8"])
def test_fused_path_determinism_full_frame(cat, name):
    """Bitwise-identical L and detections over repeated fused calls on a
    full 4096^2 frame (thousands of CTAs in flight: races would show)."""
    D = _D()
    x = torch.as_tensor(synth.config3_frame(4096)).cuda()
    runs = [D.blur_laplacian_detect(x, cat[name], return_fields=True) for _ in range(3)]
    for d, _, lap in runs[1:]:
        assert torch.equal(lap, runs[0][2])
        assert d.count == runs[0][0].count
        assert torch.equal(d.y, runs[0][0].y) and torch.equal(d.x, runs[0][0].x)


def test_derivative_field(cat, golden):
    E = _E()
    x = _f32(golden["in/rand"])
    fld = E.derivative_field(x, cat["rp4"], 3)
    B = O.blur(x, cat["rp4"])
    d1 = F.FirKernel(F.VM_BANK3[1], "anti", 1)
    d2 = F.FirKernel(F.VM_BANK3[2], "sym", 2)
    assert max_rel_err(fld[(2, 0)], O.conv_rows(B, d2)) < 1e-4
    assert max_rel_err(fld[(1, 1)], O.conv_cols(O.conv_rows(B, d1), d1)) < 1e-4
    assert set(fld.images) == {(0, 0), (1, 0), (0, 1), (2, 0), (1, 1), (0, 2)}


# ---------------------------------------------------------------------------
# the five BASELINE configs (full pipeline through vmf_blur_lap_detect)
# ---------------------------------------------------------------------------
def _check_pipeline(x, stage, frac=0.5, lap_scale=1.0, label=""):
    D = _D()
    dets, blur, lap = D.blur_laplacian_detect(x, stage, frac=frac, lap_scale=lap_scale,
                                              return_fields=True)
    B, L, (ys, xs, vs, thr) = O.pipeline(x, stage, frac=frac, lap_scale=lap_scale)
    eb, el = max_rel_err(blur, B), max_rel_err(lap, L)
    assert eb < TOL_REL, (label, "blur", eb)
    assert el < TOL_REL, (label, "laplacian", el)
    exempt, bad = compare_blobs(dets.as_set(), set(zip(ys.tolist(), xs.tolist())), L, thr)
    assert not bad, (label, bad[:10])
    assert not dets.overflow
    return dict(blur_err=eb, lap_err=el, n_ref=len(ys), n_gpu=dets.count, exempt=exempt)


def test_config1_repeated_pole(cat):
    x = synth.config1_frame()
    for name in ("rp4", "rp4_k2"):
        _check_pipeline(x, cat[name], label=f"config1/{name}")


def test_config2_fir(cat):
    x = synth.config2_frame()
    r = {}
    for name in ("sg3.2", "g4_k16"):
        r[name] = _check_pipeline(x, cat[name], label=f"config2/{name}")
    assert r["sg3.2"]["n_gpu"] > 0 and r["g4_k16"]["n_gpu"] > 0


@pytest.mark.parametrize("frac", [0.5, 0.01])
@pytest.mark.parametrize("family", ["iir", "fir"])
def test_config3_scale_space(cat, family, frac):
    """(At frac 0.5 the sigma 32 plane's edge values, which set the stack
    maximum, leave no 3x3x3 extremum in this frame; 0.01 keeps hundreds.)"""
    D = _D()
    x = synth.config3_frame(2048)  # quarter-area instance; the 4096^2 run is in bench
    spec = synth.CONFIG_STAGES[3]
    stages = [cat[n] for n in spec[family]]
    sig = spec["sigmas"]
    dets, stack = D.scale_space_detect(x, stages, sig, frac=frac, return_stack=True)
    N = np.stack([O.laplacian(O.blur(x, s)) * (g * g) for s, g in zip(stages, sig)])
    for i in range(len(sig)):
        e = max_rel_err(stack[i], N[i])
        assert e < TOL_REL, (family, sig[i], e)
    ss, ys, xs, vs, thr = O.detect3x3x3(N, frac)
    if frac < 0.1:
        assert len(ss) > 100 and dets.count > 100, (len(ss), dets.count)
    exempt, bad = compare_blobs(dets.as_set(), set(zip(ss.tolist(), ys.tolist(), xs.tolist())),
                                N, thr, stack=True)
    assert not bad, bad[:10]


@pytest.mark.parametrize("family", ["iir", "fir"])
def test_scale_space_candidates_equal_full_stack_rule(cat, family, monkeypatch):
    """The scale-space rule from the column passes' candidate lists
    (vmf_detect3x3x3_cands) returns exactly what the full-stack rule
    (vmf_detect3x3x3 over the whole stack) returns -- same detections, values,
    order and threshold -- and a list cut short falls back to the full rule."""
    D = _D()
    x = synth.config3_frame(2048)
    spec = synth.CONFIG_STAGES[3]
    stages = [cat[n] for n in spec[family]]
    sig = spec["sigmas"]
    frac = 0.01  # (the sigma 32 plane's edge values set the stack max: none clear 0.1 of it)
    fast, stack = D.scale_space_detect(x, stages, sig, frac=frac, return_stack=True)
    from paper_1912_07133_b200 import _lib, detect
    import ctypes as C
    ns, (h, w) = len(sig), x.shape
    st = torch.from_numpy(stack).cuda()
    L = _lib.lib()
    ws = torch.empty(L.vmf_detect3x3x3_workspace_bytes(ns, h, w), dtype=torch.uint8, device="cuda")
    det = torch.empty((1 << 18, 3), dtype=torch.int32, device="cuda")
    val = torch.empty(1 << 18, dtype=torch.float32, device="cuda")
    scal = torch.zeros(2, dtype=torch.int64, device="cuda")
    n_host = C.c_int64(0)
    _lib.check(L.vmf_detect3x3x3(st.data_ptr(), ns, h, w, w, h * w, frac, det.data_ptr(),
                                 val.data_ptr(), 1 << 18, scal.data_ptr(), scal.data_ptr() + 8,
                                 C.byref(n_host), ws.data_ptr(), ws.numel(),
                                 torch.cuda.current_stream().cuda_stream))
    n = n_host.value
    assert fast.count == n > 0
    assert fast.threshold == float(scal[1:2].view(torch.float32)[0].item())
    d = det[:n].cpu().numpy()
    np.testing.assert_array_equal(np.asarray(fast.s), d[:, 0])
    np.testing.assert_array_equal(np.asarray(fast.y), d[:, 1])
    np.testing.assert_array_equal(np.asarray(fast.x), d[:, 2])
    np.testing.assert_array_equal(np.asarray(fast.value), val[:n].cpu().numpy())
    monkeypatch.setattr(detect, "SS_CAND_CAP", 4)  # every list overflows: the full rule
    slow = D.scale_space_detect(x, stages, sig, frac=frac)
    assert slow.as_set() == fast.as_set() and slow.count == fast.count


def test_config4_u16_stream(cat):
    frames = synth.config4_stream(n_frames=3)
    for f in frames:
        _check_pipeline(f, cat["rp6"], label="config4")


def test_config5_coarse_scale(cat):
    x = synth.config5_frame(4096)  # quarter-area instance of the 8192^2 frame
    _check_pipeline(x, cat["bw48"], label="config5/bw48")
    _check_pipeline(x, cat["sg38.4"], label="config5/sg38.4")


def test_candidate_overflow_fallback_matches(cat, monkeypatch):
    """The ordered full-frame NMS used when a candidate buffer overflows
    (colfinal's fallback) gives the same blob list as the fast path."""
    D = _D()
    x = synth.config1_frame()
    fast = D.blur_laplacian_detect(x, cat["rp4_k2"], frac=0.3)
    monkeypatch.setenv("VMF_FORCE_FULLSCAN", "1")
    # (the full scan reads L: with the fields requested L is stored; without,
    # the candidate list covers every possible extremum and never overflows)
    slow = D.blur_laplacian_detect(x, cat["rp4_k2"], frac=0.3, return_fields=True)[0]
    assert fast.count == slow.count > 0
    np.testing.assert_array_equal(fast.y, slow.y)
    np.testing.assert_array_equal(fast.x, slow.x)
    np.testing.assert_array_equal(fast.value, slow.value)


def test_detect_sweep_matches_single_scale_calls(cat):
    """detect_sweep queues every scale without host synchronisation and reads
    all results back at once; each scale must equal the one-call path."""
    D = _D()
    x = synth.config3_frame(1024)
    names = synth.CONFIG_STAGES[3]["iir"][:3] + ["g4_k16"]
    sweep = D.detect_sweep(x, [cat[n] for n in names], frac=0.5)
    assert len(sweep) == len(names)
    for name, got in zip(names, sweep):
        ref = D.blur_laplacian_detect(x, cat[name], frac=0.5)
        assert got.count == ref.count > 0, name
        assert got.threshold == ref.threshold, name
        np.testing.assert_array_equal(got.y, ref.y)
        np.testing.assert_array_equal(got.x, ref.x)
        np.testing.assert_array_equal(got.value, ref.value)


def test_stream_detect_matches_per_frame(cat):
    """Config-4 stream front end (double-buffered uploads on a copy stream)
    gives each frame's single-call result; the first frame is also checked
    against the oracle pipeline."""
    D = _D()
    frames = synth.config4_stream(n_frames=4, size=512)
    host = torch.from_numpy(frames).pin_memory()
    got = D.stream_detect(host, cat["rp6"], frac=0.5)
    assert len(got) == 4
    for f, g in zip(frames, got):
        ref = D.blur_laplacian_detect(f, cat["rp6"], frac=0.5)
        assert g.count == ref.count
        np.testing.assert_array_equal(g.y, ref.y)
        np.testing.assert_array_equal(g.x, ref.x)
        np.testing.assert_array_equal(g.value, ref.value)
    _check_pipeline(frames[0], cat["rp6"], label="config4/stream")


@pytest.mark.parametrize("ntaps", [1, 3, 5, 7, 9, 11, 13, 15, 19, 23, 29, 41, 63, 71, 101])
def test_fir_every_tap_remainder(ntaps, monkeypatch):
    """The register-blocked FIR runs taps in blocks of 8 and the last n % 8
    taps separately (1: from the samples already in the window; 2..4: a half
    block; 5..7: a full block over zero-padded taps), with the row window
    staged in 16-byte units only when k % 4 == 0: random symmetric kernels of
    every remainder and both k parities, through the row / column leaves and
    the fused FIR column pass, against the oracle."""
    E, D = _E(), _D()
    rng = np.random.default_rng(ntaps)
    half = rng.uniform(0.1, 1.0, ntaps // 2 + 1)
    taps = np.concatenate([half[:0:-1], half])
    taps /= taps.sum()
    f = F.FirKernel(tuple(taps.tolist()), "sym", 0)
    x = rng.standard_normal((131, 1100)).astype(np.float32)
    assert max_rel_err(E.conv_rows(x, f), O.conv_rows(x, f)) < PASS_TOL, ntaps
    assert max_rel_err(E.conv_cols(x, f), O.conv_cols(x, f)) < PASS_TOL, ntaps
    y = (0.05 * rng.standard_normal((301, 517))).astype(np.float32)
    yy, xx = np.ogrid[:301, :517]
    for cy, cx in ((40, 60), (150, 300), (280, 500)):
        y += np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / 18.0).astype(np.float32)
    _check_pipeline(y, f, label=f"fir {ntaps} taps")  # (tensor cores from 33 taps)
    monkeypatch.setenv("VMF_NO_FIRTC", "1")  # the fp64 fused FIR column pass at every length
    _check_pipeline(y, f, label=f"fir {ntaps} taps (fp64 fused pass)")


def test_fir_fused_long_taps(cat):
    """385-tap colored SG (config 5's FIR) on the fused FIR column pass."""
    x = synth.config5_frame(1024)
    _check_pipeline(x, cat["sg38.4"], label="config5/sg38.4 fused")


@pytest.mark.parametrize("lpf", ["g3", "rp4"])
def test_derivative_field_fused(cat, golden, lpf):
    """derivative_field with a FIR blur takes the fused pass (all six images
    from the fp64 blur) and matches the oracle's bank."""
    E = _E()
    x = _f32(golden["in/rand"])
    g = F.gaussian_fir(3.0, 0, 15) if lpf == "g3" else cat[lpf]
    fld = E.derivative_field(x, g, 3)
    B = O.blur(x, g)
    d1 = F.FirKernel(F.VM_BANK3[1], "anti", 1)
    d2 = F.FirKernel(F.VM_BANK3[2], "sym", 2)
    ref = {(0, 0): B, (1, 0): O.conv_rows(B, d1), (0, 1): O.conv_cols(B, d1),
           (2, 0): O.conv_rows(B, d2), (0, 2): O.conv_cols(B, d2),
           (1, 1): O.conv_cols(O.conv_rows(B, d1), d1)}
    assert set(fld.images) == set(ref)
    for k, v in ref.items():
        assert max_rel_err(fld[k], v) < 1e-5, k


@pytest.mark.parametrize("shape", [(67, 131), (300, 517), (129, 64), (1000, 33), (33, 1000)])
@pytest.mark.parametrize("name", ["rp4", "rp4_k2", "g2_k8"])
def test_fused_path_odd_shapes(cat, shape, name):
    """Odd / ragged shapes through the fused path (row-pass fallback widths,
    partial bands and column tiles, short images) against the oracle."""
    # seed from the parameters (crc32: str hashes are salted per process)
    rng = np.random.default_rng(zlib.crc32(repr((shape, name)).encode()) & 0xFFFF)
    h, w = shape
    x = (0.05 * rng.standard_normal((h, w))).astype(np.float32)
    for _ in range(6):  # a few blobs so the threshold selects something
        cy, cx = rng.integers(0, h), rng.integers(0, w)
        yy, xx = np.ogrid[:h, :w]
        x += np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / 18.0).astype(np.float32)
    _check_pipeline(x, cat[name], label=f"{name} {shape}")


@pytest.mark.parametrize("seed", [38610, 43228, 55631, 62877])
def test_negative_maximum_is_not_a_blob(cat, seed):
    """A strict local MAXIMUM whose value is negative (a shallow spot inside a
    dark region) has |L| >= t but is not a blob: the rule is L >= t for
    maxima and -L >= t for minima.  These seeds (found by
    tools/repro_odd.py over 65536 inputs) put one at column W-2 of a 1000x33
    frame."""
    h, w = 1000, 33
    rng = np.random.default_rng(seed)
    x = (0.05 * rng.standard_normal((h, w))).astype(np.float32)
    for _ in range(6):
        cy, cx = rng.integers(0, h), rng.integers(0, w)
        yy, xx = np.ogrid[:h, :w]
        x += np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / 18.0).astype(np.float32)
    _check_pipeline(x, cat["rp4"], label=f"rp4 seed {seed}")


def test_stream_sweep_matches_detect_sweep(cat):
    """The overlapped multi-scale frame stream gives each frame the results
    of a detect_sweep call, including sets larger than the per-frame
    readback (d2h_cap) and a device-resident frame."""
    D = _D()
    frames = [f.astype(np.float32) for f in synth.config4_stream(n_frames=3, size=512)]
    stages = [cat[n] for n in ("rp2", "rp4", "g2_k8")]
    host = [torch.from_numpy(f).pin_memory() for f in frames]
    got = D.stream_sweep(host, stages, d2h_cap=8)
    dev = D.stream_sweep([host[0].cuda()], stages, d2h_cap=8)[0]
    assert len(got) == 3
    for f, g in zip(frames, got):
        ref = D.detect_sweep(f, stages)
        assert len(g) == len(ref) == 3
        for a, b in zip(g, ref):
            assert a.count == b.count and a.threshold == b.threshold
            np.testing.assert_array_equal(a.y, b.y)
            np.testing.assert_array_equal(a.x, b.x)
            np.testing.assert_array_equal(a.value, b.value)
    for a, b in zip(dev, got[0]):
        np.testing.assert_array_equal(a.value, b.value)
    assert max(d.count for d in got[0]) > 8


def test_derivative_field_order5(cat):
    """Higher-order bank (fir_vm_bank(5), taps from the reference-generated
    design golden file) through the unfused path; order 1 is rejected like
    the reference's fir_vm_bank."""
    import json
    import os

    E = _E()
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "design_golden.json")))
    bank = [k["taps"] for k in g["fir_vm_bank(5, 2, 'behind_blur')"]["fir"]]
    x = _f32(synth.config1_frame())[:200, :256]
    st = cat["g2_k8"]
    got = E.derivative_field(x, st, order=5)
    ref = O.derivative_field(x, st, order=5, bank=bank)
    assert set(got.images) == set(ref)
    for key, r in ref.items():
        # derivatives of total order >= 4 are differences of the fp32-rounded
        # blur (the fused order-3 bank works on the fp64 blur): 1e-3 there
        tol = 1e-4 if sum(key) <= 3 else 1e-3
        assert max_rel_err(got[key], r) < tol, key
    with pytest.raises(ValueError):
        E.derivative_field(x, st, order=1)


@pytest.mark.parametrize("shape", [(257, 389), (70, 1030), (1024, 131)])
@pytest.mark.parametrize("name", ["rp4_k2", "rp8", "rp4_k4", "bw6", "g4_k16", "g16_k64"])
def test_column_leaves_fast_paths(cat, shape, name):
    """iir_cols / conv_cols on fp32 frames run on the fused pipeline's column
    kernels in blur-only mode (colapply / firapply MODE 3); odd shapes, both
    parities of band and tile edges."""
    E = _E()
    st = cat[name]
    if F.is_fir(st) and len(st.taps) > shape[0]:
        pytest.skip("kernel longer than the column")
    x = np.random.default_rng(11).standard_normal(shape).astype(np.float32) + 0.5
    op = "conv_cols" if F.is_fir(st) else "iir_cols"
    got = getattr(E, op)(x, st)
    want = getattr(O, op)(x, st)
    assert max_rel_err(got, want) < PASS_TOL, (name, shape)


def test_scale_sharded_detect_single_rank(cat):
    """shard.scale_space_detect on one rank (no process group) equals the
    unsharded scale-space detector: same L stack, threshold and blobs (the
    multi-rank exchange logic is covered on CPU by test_multiproc.py)."""
    from paper_1912_07133_b200 import shard

    D = _D()
    x = synth.config3_frame(1024)
    spec = synth.CONFIG_STAGES[3]
    stages = [cat[n] for n in spec["iir"]]
    sig = spec["sigmas"]
    ref = D.scale_space_detect(x, stages, sig, frac=0.5)
    got = shard.scale_space_detect(x, stages, sig, frac=0.5)
    assert got.threshold == ref.threshold and got.count == ref.count
    assert got.as_set() == ref.as_set()
