"""Parity helpers (BASELINE.json north_star): responses within 1e-4 of the
per-frame max |response|; blob sets identical except near-ties -- candidates
whose response is within that tolerance of the threshold or of a
neighbour."""
import numpy as np

TOL_REL = 1e-4


def max_rel_err(got, want):
    want = np.asarray(want, dtype=np.float64)
    scale = np.abs(want).max()
    return float(np.abs(np.asarray(got, dtype=np.float64) - want).max() / (scale or 1.0))


def _near_tie(L, pt, thr, tol, stack=False):
    if stack:
        s, y, x = pt
        P = L[s]
    else:
        y, x = pt
        P = L
    v = P[y, x]
    if abs(abs(v) - thr) < tol:
        return True
    h, w = P.shape
    planes = [P]
    if stack:
        planes += [L[t] for t in (s - 1, s + 1) if 0 <= t < L.shape[0]]
    for Q in planes:
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                yy, xx = min(max(y + dy, 0), h - 1), min(max(x + dx, 0), w - 1)
                if Q is P and yy == y and xx == x:
                    continue
                if abs(Q[yy, xx] - v) < tol:
                    return True
    return False


def compare_blobs(got_set, want_set, L_ref, thr_ref, stack=False, tol_rel=TOL_REL):
    """-> (n_exempt, offending list).  Offending must be empty."""
    L_ref = np.asarray(L_ref, dtype=np.float64)
    tol = tol_rel * np.abs(L_ref).max()
    diff = got_set ^ want_set
    bad = [p for p in diff if not _near_tie(L_ref, p, thr_ref, tol, stack)]
    return len(diff) - len(bad), bad
