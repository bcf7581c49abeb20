"""Pin the CPU oracle (oracle/vmf_oracle.c) against golden vectors produced
by the live reference (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1912_07133_b200 import filters as F


def _items(golden, prefix):
    return [(k, v) for k, v in golden.items() if k.startswith(prefix)]


@pytest.mark.parametrize("op", ["iir_rows", "iir_cols", "conv_rows", "conv_cols"])
def test_oracle_matches_reference_kernels(golden, cat, op):
    fn = getattr(O, op)
    items = _items(golden, op + "/")
    assert items
    for key, want in items:
        _, fname, iname = key.split("/")
        got = fn(golden[f"in/{iname}"], cat[fname])
        # same operation order, no FMA contraction -> bit-identical to numba
        np.testing.assert_array_equal(got, want, err_msg=key)


def test_oracle_blur_matches_reference(golden, cat):
    for key, want in _items(golden, "blur/"):
        _, fname, iname = key.split("/")
        np.testing.assert_array_equal(O.blur(golden[f"in/{iname}"], cat[fname]), want,
                                      err_msg=key)


def test_oracle_laplacian_matches_derivative_field(golden, cat):
    for fname in ("rp4", "g1.5_k8", "bw6"):
        for iname in ("rand", "f32"):
            B = O.blur(golden[f"in/{iname}"], cat[fname])
            want = golden[f"field/{fname}/{iname}/20"] + golden[f"field/{fname}/{iname}/02"]
            np.testing.assert_array_equal(O.laplacian(B), want)
            # the bank's other members through the oracle's conv (engine.py:218-227)
            d1 = F.FirKernel(F.VM_BANK3[1], "anti", 1)
            np.testing.assert_array_equal(O.conv_rows(B, d1), golden[f"field/{fname}/{iname}/10"])
            np.testing.assert_array_equal(O.conv_cols(B, d1), golden[f"field/{fname}/{iname}/01"])
            np.testing.assert_array_equal(O.conv_cols(O.conv_rows(B, d1), d1),
                                          golden[f"field/{fname}/{iname}/11"])


def test_oracle_thread_count_does_not_change_output(golden, cat):
    # analogue of tests/test_engine.py:119-128
    x = golden["in/rand"]
    O.set_threads(1)
    a = O.blur(x, cat["rp4"]), O.blur(x, cat["g4_k16"])
    O.set_threads(7)
    b = O.blur(x, cat["rp4"]), O.blur(x, cat["g4_k16"])
    O.set_threads(0)
    for u, v in zip(a, b):
        np.testing.assert_array_equal(u, v)


def test_detect_restatements_agree():
    rng = np.random.default_rng(5)
    for shape in ((37, 53), (3, 3), (1, 9), (64, 64)):
        L = rng.standard_normal(shape)
        L[rng.random(shape) < 0.1] = 0.25  # plateaus: ties must not count
        for frac in (0.0, 0.3, 0.5):
            a = O.detect3x3(L, frac)
            b = O.detect3x3_np(L, frac)
            np.testing.assert_array_equal(a[0], b[0])
            np.testing.assert_array_equal(a[1], b[1])
            np.testing.assert_array_equal(a[2], b[2])


def test_detect_edge_semantics():
    L = np.zeros((5, 5))
    L[0, 2] = 9.0     # border: never a strict extremum under replicate edges
    L[2, 2] = 5.0     # interior maximum
    L[3, 3] = -4.0    # interior minimum (< 0.5 * max |L| = 4.5 -> dropped)
    ys, xs, vs, thr = O.detect3x3(L, 0.5)
    assert thr == 4.5
    assert list(zip(ys, xs)) == [(2, 2)]
    ys, xs, vs, thr = O.detect3x3(L, 0.4)
    assert list(zip(ys, xs)) == [(2, 2), (3, 3)]


def test_detect3x3x3_one_sided_and_strict():
    rng = np.random.default_rng(9)
    N = rng.standard_normal((3, 12, 12)) * 0.01
    N[0, 5, 5] = 1.0       # first scale: compared with scale 1 only
    N[1, 5, 5] = 0.9       # not an extremum across scales (0 has 1.0)
    N[2, 8, 3] = -1.0
    ss, ys, xs, vs, thr = O.detect3x3x3(N, 0.5)
    assert list(zip(ss, ys, xs)) == [(0, 5, 5), (2, 8, 3)]


def test_gaussian_fir_restatement(golden):
    for key, want in _items(golden, "gauss/"):
        _, s, d, k = key.split("/")
        got = F.gaussian_fir(float(s), int(d), int(k)).taps
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-15)


def test_catalog_filters_are_valid_blurs(cat):
    from paper_1912_07133_b200.engine import stability_margin

    for name, f in cat.items():
        if F.is_iir(f):
            assert stability_margin(f) > 0, name
            # dc gain b0 + 2 * sum(b)/(1+sum(a)) == 1 for blurs
            g = f.b_zero + 2 * sum(f.b_plus) / (1 + sum(f.a_plus))
            assert abs(g - 1.0) < 1e-9, name
        elif not name.startswith("vm_bank"):
            assert abs(sum(f.taps) - 1.0) < 1e-12, name


def test_strict_extrema_bound_sizes_the_candidate_list():
    """The fp32 column pass sizes its candidate list for 2 ceil(h/2) ceil(w/2)
    entries (vmf_colpass32.cu cand32_capacity) so that, with L kept in its
    tiles, no overflow can occur: strict 3x3 maxima are pairwise more than
    one pixel apart (a 2x2 block holds at most one), and so are the minima.
    Checked at threshold 0 on the densest patterns and on noise."""
    rng = np.random.default_rng(7)
    for h, w in [(8, 8), (9, 7), (64, 64), (33, 65)]:
        bound = 2 * (-(-h // 2)) * (-(-w // 2))
        yy, xx = np.mgrid[0:h, 0:w]
        pats = [
            rng.standard_normal((h, w)),
            ((yy % 2 == 0) & (xx % 2 == 0)).astype(float) - ((yy % 2 == 1) & (xx % 2 == 1)),
            np.cos(np.pi * yy) * np.cos(np.pi * xx),
        ]
        for a in pats:
            ys, xs, vs, thr = O.detect3x3_np(a, thr=0.0)
            assert len(ys) <= bound, (h, w, len(ys), bound)
            # maxima alone and minima alone each fit a quarter
            mx = [(y, x) for y, x in zip(ys, xs) if all(
                a[y, x] > a[min(max(y + i, 0), h - 1), min(max(x + j, 0), w - 1)]
                for i in (-1, 0, 1) for j in (-1, 0, 1) if i or j)]
            assert len(mx) <= (-(-h // 2)) * (-(-w // 2))
