"""Fused hot path: blur (rows, columns) -> Laplacian -> threshold + NMS.

This is the north-star pipeline (BASELINE.json): stage 1/2 blur, stage 3
Laplacian L = D20 + D02 (engine.py:215-227, blob.py:161) and stage 4
detection.  The reference has no Laplacian + 3x3-NMS detector; the rule is
the restatement of SURVEY.md §8(d) (conventions from blob.py:162-168):

* single scale: keep (y, x) iff L(y, x) is strictly greater (smaller) than
  its 8 edge-replicated neighbours and L >= t (-L >= t), t = frac * max|L|;
* scale space (config 3): N_s = sigma_s^2 L_s; strict against the 8
  in-scale and 9 + 9 adjacent-scale neighbours (one-sided at the ends);
  t = frac * max over the whole stack of |N|.

Detections come back sorted by (y, x) (and scale first for the stack).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .engine import (_as_image, _dptr, _fir_checks, _iir_checks, _pitch, _ptr, _sign, _stream,
                     _workspace)
from .filters import is_fir, is_iir

__all__ = ["Detections", "make_stage", "blur_laplacian_detect", "detect_sweep",
           "scale_space_detect", "stream_detect", "stream_sweep",
           "pgm_stream_detect"]


@dataclass
class Detections:
    """Blob list.  `s` is the scale index (scale-space detection only)."""

    y: object
    x: object
    value: object
    threshold: float
    count: int            # total number of detections found
    overflow: bool        # True if count > capacity (list truncated)
    s: object = None

    def __len__(self):
        return int(len(self.y))

    def as_set(self):
        ys = np.asarray(_np(self.y)).tolist()
        xs = np.asarray(_np(self.x)).tolist()
        if self.s is None:
            return set(zip(ys, xs))
        return set(zip(np.asarray(_np(self.s)).tolist(), ys, xs))


def _np(t):
    return t.cpu().numpy() if isinstance(t, torch.Tensor) else t


class _Stage:
    """A vmf_stage plus the ctypes arrays it points into (kept alive)."""

    def __init__(self, stage):
        self.src = stage
        self.s = _lib.VmfStage()
        if is_fir(stage):
            self._taps = _dptr(stage.taps)
            self.s.kind, self.s.n = _lib.VMF_STAGE_FIR, len(stage.taps)
            self.s.taps = C.cast(self._taps, C.POINTER(C.c_double))
        elif is_iir(stage):
            self._b, self._a = _dptr(stage.b_plus), _dptr(stage.a_plus)
            self.s.kind, self.s.n = _lib.VMF_STAGE_IIR, len(stage.a_plus)
            self.s.b_plus = C.cast(self._b, C.POINTER(C.c_double))
            self.s.a_plus = C.cast(self._a, C.POINTER(C.c_double))
            self.s.b_zero, self.s.sign = float(stage.b_zero), _sign(stage)
        else:
            raise TypeError(f"unsupported stage type {type(stage).__name__}")

    def check(self, length: int):
        if is_fir(self.src):
            _fir_checks(self.src, length)
        else:
            _iir_checks(self.src, length)


def make_stage(stage) -> _Stage:
    return _Stage(stage)


def _fused(x, code, row: _Stage, col: _Stage, lap_scale, frac, blur_out, lap_out, cap, sync,
           out=None, slot: int = 0):
    """One vmf_blur_lap_detect call.  `out` = preallocated (det_yx [cap, 2],
    det_val [cap], scal [2]) device tensors; with sync=False nothing waits
    for the GPU and the count is read from scal[0] later."""
    h, w = x.shape
    row.check(w)
    col.check(h)
    L = _lib.lib()
    nbytes = L.vmf_blur_lap_detect_workspace_bytes(h, w, C.byref(row.s), C.byref(col.s))
    ws = _workspace(nbytes, slot)
    dev = x.device
    cap = int(cap)
    if out is None:
        det_yx = torch.empty((max(cap, 1), 2), dtype=torch.int32, device=dev)
        det_val = torch.empty((max(cap, 1),), dtype=torch.float32, device=dev)
        scal = torch.empty(2, dtype=torch.int64, device=dev)  # [n_det, thr(float bits)]
    else:
        det_yx, det_val, scal = out
    n_host = C.c_int64(0)
    _lib.check(L.vmf_blur_lap_detect(
        _ptr(x), code, h, w, _pitch(x), C.byref(row.s), C.byref(col.s), float(lap_scale),
        float(frac), _ptr(blur_out) if blur_out is not None else None,
        _ptr(lap_out) if lap_out is not None else None, _ptr(det_yx), _ptr(det_val), cap,
        _ptr(scal), scal.data_ptr() + 8, C.byref(n_host) if sync else None, _ptr(ws),
        ws.numel(), _stream()))
    return det_yx, det_val, scal, n_host.value


# scales (or frames) in flight on the per-scale fused path (measured on B200:
# 1 -> 0.617 ms, 3 -> 0.532 ms per 5-scale sweep); VMF_SWEEP_STREAMS overrides
# it for experiments
SWEEP_STREAMS = int(os.environ.get("VMF_SWEEP_STREAMS", "3"))
# the multi-scale sweep's column passes: one stream per scale, up to this many
# (5 scales: 3 streams 0.433 ms, 4: 0.435, 5: 0.416 -- with fewer streams a
# stream's second scale waits behind the first's latency-bound finaliser);
# VMF_SWEEP_SCALE_STREAMS overrides it
SWEEP_SCALE_STREAMS = int(os.environ.get("VMF_SWEEP_SCALE_STREAMS", "8"))
_side_streams: dict = {}


def _side(n: int):
    lst = _side_streams.setdefault(torch.cuda.current_device(), [])
    while len(lst) < n:
        lst.append(torch.cuda.Stream())
    return lst[:n]


_SWEEP_SLOT = 1000  # workspace slot of the multi-scale row pass's outputs


def _sweep_ok(x, code, stages) -> bool:
    """The multi-scale fp32 path takes this sweep (vmf_sweep_supported)."""
    if isinstance(x, (list, tuple)) or code != _lib.VMF_F32 or not stages:
        return False
    if os.environ.get("VMF_NO_SWEEP"):
        return False
    h, w = x.shape
    arr = (_lib.VmfStage * len(stages))(*[st.s for st in stages])
    return bool(_lib.lib().vmf_sweep_supported(_ptr(x), code, h, w, _pitch(x), len(stages), arr,
                                               arr))


# scales per row pass of a sweep: the column passes of one group overlap the
# next group's row pass (VMF_SWEEP_GROUP overrides it for experiments)
SWEEP_GROUP = int(os.environ.get("VMF_SWEEP_GROUP", "5"))


def _sweep_launch_multi(x, code, stages, frac, lap_scales, cap, outs, laps, conc):
    """Row passes for groups of scales (vmf_sweep_rows: the Laplacian of the
    frame and its staging shared by a group's scales), each followed by its
    scales' column passes on `conc` side streams (vmf_sweep_detect) that
    overlap the next group's row pass."""
    L = _lib.lib()
    h, w = x.shape
    ns = len(stages)
    grp = max(1, min(SWEEP_GROUP, 5))
    cur = torch.cuda.current_stream()
    side = _side(conc) if conc > 1 else [cur]
    k = 0
    for g0 in range(0, ns, grp):
        sub = stages[g0:g0 + grp]
        ng = len(sub)
        arr = (_lib.VmfStage * ng)(*[st.s for st in sub])
        sws = _workspace(L.vmf_sweep_workspace_bytes(h, w, ng), _SWEEP_SLOT + g0)
        _lib.check(L.vmf_sweep_rows(_ptr(x), code, h, w, _pitch(x), ng, arr, arr, _ptr(sws),
                                    sws.numel(), _stream()))
        if conc > 1:
            for s in side:
                s.wait_stream(cur)
        for j in range(ng):
            i = g0 + j
            sc = 1.0 if lap_scales is None else float(lap_scales[i])
            det_yx, det_val, scal = outs[i]
            st_ = side[k % len(side)]
            k += 1
            with torch.cuda.stream(st_):
                ws = _workspace(L.vmf_sweep_detect_workspace_bytes(h, w, C.byref(stages[i].s)),
                                1 + (k - 1) % len(side))
                lap = None if laps is None else laps[i]
                _lib.check(L.vmf_sweep_detect(
                    j, h, w, ng, C.byref(stages[i].s), sc, float(frac),
                    _ptr(lap) if lap is not None else None, _ptr(det_yx), _ptr(det_val), int(cap),
                    _ptr(scal), scal.data_ptr() + 8, _ptr(sws), sws.numel(), _ptr(ws), ws.numel(),
                    _stream()))
    if conc > 1:
        for s in side:
            cur.wait_stream(s)


def _sweep_launch(x, code, stages, frac, lap_scales, cap, outs, laps=None, conc=None):
    """Queue one fused single-scale pass per stage.  The scales of a sweep
    are independent (same frame, own outputs), so with conc > 1 they run on
    `conc` side streams, each with its own workspace slot, forked from and
    joined back into the current stream: one scale's latency-bound phases
    (band scan, finaliser, kernel tails) overlap another's row pass.  When
    the fp32 path takes the sweep, one row pass serves every scale."""
    ns = len(stages)
    if _sweep_ok(x, code, stages):
        conc = max(1, min(int(SWEEP_SCALE_STREAMS if conc is None else conc), ns))
        _sweep_launch_multi(x, code, stages, frac, lap_scales, cap, outs, laps, conc)
        return
    conc = max(1, min(int(SWEEP_STREAMS if conc is None else conc), ns))

    def one(i, slot):  # x: one frame for every stage, or a list (one frame per stage)
        sc = 1.0 if lap_scales is None else float(lap_scales[i])
        xi = x[i] if isinstance(x, (list, tuple)) else x
        _fused(xi, code, stages[i], stages[i], sc, frac, None, None if laps is None else laps[i],
               cap, False, out=outs[i], slot=slot)

    if conc == 1:
        for i in range(ns):
            one(i, 0)
        return
    cur = torch.cuda.current_stream()
    side = _side(conc)
    for s in side:
        s.wait_stream(cur)
    for i in range(ns):
        with torch.cuda.stream(side[i % conc]):
            one(i, 1 + i % conc)
    for s in side:
        cur.wait_stream(s)


def blur_laplacian_detect(img, lpf, frac: float = 0.5, col_stage=None, lap_scale: float = 1.0,
                          cap: int = 1 << 18, return_fields: bool = False):
    """Whole north-star path in one native call (vmf_blur_lap_detect).

    img: 2-D numpy array / torch tensor (fp32 or uint16).  lpf: the blur
    stage (FirKernel or ThreePartIIR; `col_stage` defaults to the same).
    Returns Detections (numpy if img was numpy) and, with return_fields,
    (blur, laplacian) as well."""
    x, kind, code = _as_image(img)
    h, w = x.shape
    row, col = _Stage(lpf), _Stage(col_stage if col_stage is not None else lpf)
    blur = lap = None
    if return_fields:
        blur = torch.empty((h, w), dtype=torch.float32, device=x.device)
        lap = torch.empty((h, w), dtype=torch.float32, device=x.device)
    det_yx, det_val, scal, n = _fused(x, code, row, col, lap_scale, frac, blur, lap, cap, True)
    thr = float(scal[1:2].view(torch.float32)[0].item()) if frac > 0 else float("nan")
    m = min(n, cap)
    yx, val = det_yx[:m], det_val[:m]
    if kind == "numpy":
        yx, val = yx.cpu().numpy(), val.cpu().numpy()
        if return_fields:
            blur, lap = blur.cpu().numpy(), lap.cpu().numpy()
    dets = Detections(yx[:, 0], yx[:, 1], val, thr, n, n > cap)
    if return_fields:
        return dets, blur, lap
    return dets


def detect_sweep(img, stages, frac: float = 0.5, lap_scales=None, cap: int = 1 << 18):
    """One frame through the fused single-scale path once per blur stage
    (config 3's IIR-vs-FIR scale sweep): the frame is uploaded once, the
    scales are queued without host synchronisation on SWEEP_STREAMS
    concurrent streams, and the detections of every scale come back in one
    device-to-host copy.
    Returns a list of Detections (numpy arrays)."""
    x, kind, code = _as_image(img)
    ns = len(stages)
    if ns == 0:
        return []
    dev = x.device
    cap = max(int(cap), 1)
    det_yx = torch.empty((ns, cap, 2), dtype=torch.int32, device=dev)
    det_val = torch.empty((ns, cap), dtype=torch.float32, device=dev)
    scal = torch.empty((ns, 2), dtype=torch.int64, device=dev)
    stg = [st if isinstance(st, _Stage) else _Stage(st) for st in stages]
    _sweep_launch(x, code, stg, frac, lap_scales, cap,
                  [(det_yx[i], det_val[i], scal[i]) for i in range(ns)])
    head = scal.cpu()                                   # counts + thresholds
    ns_det = head[:, 0].tolist()
    thr = head[:, 1:2].contiguous().view(torch.float32)[:, 0].tolist()
    mmax = min(max(ns_det), cap)
    yx = det_yx[:, :mmax].cpu().numpy()
    val = det_val[:, :mmax].cpu().numpy()
    out = []
    for i in range(ns):
        n = int(ns_det[i])
        m = min(n, cap)
        out.append(Detections(yx[i, :m, 0], yx[i, :m, 1], val[i, :m], float(thr[i]), n, n > cap))
    return out


SS_CAND_CAP = 1 << 16  # per-scale candidate list of the scale-space rule


def _scale_space_launch(x, code, stages, sigmas, frac, stack, cands, det, val, scal):
    """Device part of scale_space_detect (frac > 0): the sweep writes each
    scale's plane of the sigma^2-normalised stack and lists its strict 3x3
    extrema above frac * that plane's max (the fused column pass's own
    detection), then vmf_detect3x3x3_cands keeps the candidates that clear
    the adjacent planes and the stack threshold.  scal[0] = -1 means a list
    was cut short (the caller runs the full-stack rule)."""
    ns = len(stages)
    h, w = x.shape
    cyx, cval, cscal = cands
    _sweep_launch(x, code, stages, frac, [float(sg) ** 2 for sg in sigmas], cyx.shape[1],
                  [(cyx[s], cval[s], cscal[s]) for s in range(ns)],
                  laps=[stack[s] for s in range(ns)])
    _lib.check(_lib.lib().vmf_detect3x3x3_cands(
        _ptr(stack), ns, h, w, w, h * w, _ptr(cyx), _ptr(cval), cyx.shape[1], _ptr(cscal),
        _ptr(det), _ptr(val), det.shape[0], _ptr(scal), scal.data_ptr() + 8, _stream()))


def scale_space_detect(img, stages, sigmas, frac: float = 0.5, cap: int = 1 << 18,
                       return_stack: bool = False):
    """Config-3 scale sweep: per scale the fused blur + Laplacian with
    lap_scale = sigma^2 into one stack, then 3x3x3 NMS over the stack
    (frac > 0: from the column passes' own candidate lists; else, and when a
    list overflows, over the whole stack)."""
    if len(stages) != len(sigmas) or not stages:
        raise ValueError("need one stage per sigma")
    x, kind, code = _as_image(img)
    h, w = x.shape
    ns = len(stages)
    stg = [_Stage(st) for st in stages]
    stack = torch.empty((ns, h, w), dtype=torch.float32, device=x.device)
    cap = int(cap)
    det = torch.empty((max(cap, 1), 3), dtype=torch.int32, device=x.device)
    val = torch.empty((max(cap, 1),), dtype=torch.float32, device=x.device)
    scal = torch.zeros(2, dtype=torch.int64, device=x.device)
    L = _lib.lib()
    n = -1
    if frac > 0:
        cands = (torch.empty((ns, SS_CAND_CAP, 2), dtype=torch.int32, device=x.device),
                 torch.empty((ns, SS_CAND_CAP), dtype=torch.float32, device=x.device),
                 torch.empty((ns, 2), dtype=torch.int64, device=x.device))
        _scale_space_launch(x, code, stg, sigmas, float(frac), stack, cands, det, val, scal)
        n = int(scal[0].item())
    if n < 0:  # the full-stack rule
        if frac <= 0:
            dummy = [(torch.empty((1, 2), dtype=torch.int32, device=x.device),
                      torch.empty(1, dtype=torch.float32, device=x.device),
                      torch.empty(2, dtype=torch.int64, device=x.device)) for _ in range(ns)]
            _sweep_launch(x, code, stg, 0.0, [float(sg) ** 2 for sg in sigmas], 0, dummy,
                          laps=[stack[s] for s in range(ns)])
        nbytes = L.vmf_detect3x3x3_workspace_bytes(ns, h, w)
        ws = _workspace(nbytes)
        n_host = C.c_int64(0)
        _lib.check(L.vmf_detect3x3x3(_ptr(stack), ns, h, w, w, h * w, float(frac), _ptr(det),
                                     _ptr(val), cap, _ptr(scal), scal.data_ptr() + 8,
                                     C.byref(n_host), _ptr(ws), ws.numel(), _stream()))
        n = n_host.value
    thr = float(scal[1:2].view(torch.float32)[0].item())
    m = min(n, cap)
    d, v = det[:m], val[:m]
    if kind == "numpy":
        d, v = d.cpu().numpy(), v.cpu().numpy()
    dets = Detections(d[:, 1], d[:, 2], v, thr, n, n > cap, s=d[:, 0])
    if return_stack:
        return dets, (stack.cpu().numpy() if kind == "numpy" else stack)
    return dets


def stream_detect(frames, stage, frac: float = 0.5, cap: int = 1 << 16):
    """Config-4 stream front end: a frame stream (n, h, w) of uint16, uint8
    or float32 in host memory (pin it for full speed) through the fused
    single-scale path.  Two device frame buffers: the upload of frame i+1
    runs on a copy stream while frame i is filtered on the current stream;
    nothing waits for the host until the end, when every frame's detections
    come back in one copy.  Returns a list of Detections, one per frame."""
    if isinstance(frames, np.ndarray):
        frames = torch.from_numpy(np.ascontiguousarray(frames))
    if frames.ndim != 3 or frames.shape[0] < 1:
        raise ValueError("frames must be an (n, h, w) array")
    if frames.dtype not in (torch.uint16, torch.uint8, torch.float32):
        frames = frames.to(torch.float32)
    n, h, w = frames.shape
    code = {torch.uint16: _lib.VMF_U16, torch.uint8: _lib.VMF_U8}.get(frames.dtype, _lib.VMF_F32)
    stg = stage if isinstance(stage, _Stage) else _Stage(stage)
    res = _StreamResults(n, cap)
    if frames.is_cuda:  # device-resident frames: SWEEP_STREAMS frames in flight
        conc = max(1, min(SWEEP_STREAMS, n))
        cur = torch.cuda.current_stream()
        side = _side(conc)
        for s in side:
            s.wait_stream(cur)
        for i in range(n):
            with torch.cuda.stream(side[i % conc]):
                _fused(frames[i], code, stg, stg, 1.0, frac, None, None, res.cap, False,
                       out=res.out(i), slot=1 + i % conc)
        for s in side:
            cur.wait_stream(s)
        return res.collect()
    up = _Uploader((h, w), frames.dtype)
    for i in range(n):
        _fused(up.put(frames[i]), code, stg, stg, 1.0, frac, None, None, res.cap, False,
               out=res.out(i))
        up.release()
    return res.collect()


class _StreamResults:
    """Device-side detection buffers of a frame stream, read back once."""

    def __init__(self, n, cap):
        dev = torch.device("cuda", torch.cuda.current_device())
        self.n, self.cap = n, max(int(cap), 1)
        self.det_yx = torch.empty((n, self.cap, 2), dtype=torch.int32, device=dev)
        self.det_val = torch.empty((n, self.cap), dtype=torch.float32, device=dev)
        self.scal = torch.empty((n, 2), dtype=torch.int64, device=dev)

    def out(self, i):
        return self.det_yx[i], self.det_val[i], self.scal[i]

    def collect(self):
        head = self.scal.cpu()
        counts = head[:, 0].tolist()
        thr = head[:, 1:2].contiguous().view(torch.float32)[:, 0].tolist()
        mmax = min(max(counts), self.cap)
        yx = self.det_yx[:, :mmax].cpu().numpy()
        val = self.det_val[:, :mmax].cpu().numpy()
        out = []
        for i in range(self.n):
            c = int(counts[i])
            m = min(c, self.cap)
            out.append(Detections(yx[i, :m, 0], yx[i, :m, 1], val[i, :m], float(thr[i]), c,
                                  c > self.cap))
        return out


class _Uploader:
    """Two device frame buffers fed by copy streams: put() enqueues the
    upload of the next host frame (waiting only for the filter of the frame
    two back) and makes the current stream wait for it; release() marks the
    buffer free once the work queued on the current stream is done.  A frame
    is uploaded as `nsplit` row blocks alternating over two copy streams
    (two DMA engines in flight: ~10 % more PCIe bandwidth than one copy)."""

    def __init__(self, shape, dtype, nsplit=None):
        dev = torch.device("cuda", torch.cuda.current_device())
        self.comp = torch.cuda.current_stream()
        self.copies = [torch.cuda.Stream(), torch.cuda.Stream()]
        self.bufs = [torch.empty(shape, dtype=dtype, device=dev) for _ in range(2)]
        self.ready = [[torch.cuda.Event() for _ in self.copies] for _ in range(2)]
        self.free = [torch.cuda.Event() for _ in range(2)]
        for e in self.free:
            e.record(self.comp)
        if nsplit is None:  # split only large frames (measured: 8 MiB frames lose ~6 % split in 4)
            nbytes = shape[0] * shape[1] * torch.empty((), dtype=dtype).element_size()
            nsplit = 4 if nbytes >= (32 << 20) else 1
        self.nsplit = max(1, min(int(nsplit), shape[0]))
        self.i = -1

    def put(self, host, after_copy=None):
        self.i += 1
        b = self.i & 1
        h = host.shape[0]
        bounds = [h * k // self.nsplit for k in range(self.nsplit + 1)]
        for c, s in enumerate(self.copies):
            s.wait_event(self.free[b])  # frame i-2 has been filtered
        for k in range(self.nsplit):
            s = self.copies[k & 1]
            with torch.cuda.stream(s):
                self.bufs[b][bounds[k]:bounds[k + 1]].copy_(host[bounds[k]:bounds[k + 1]],
                                                           non_blocking=True)
        for c, s in enumerate(self.copies):
            self.ready[b][c].record(s)
            self.comp.wait_event(self.ready[b][c])
        if after_copy is not None:  # host buffer reusable once both copies are done
            self.copies[0].wait_event(self.ready[b][1])
            after_copy.record(self.copies[0])
        return self.bufs[b]

    def release(self):
        b = self.i & 1
        self.bufs[b].record_stream(self.comp)
        self.free[b].record(self.comp)


_pinned_cache: dict = {}


def _pinned(tag: str, shape, dtype) -> torch.Tensor:
    """Grow-only pinned host buffers for readbacks: a fresh pinned
    allocation (cudaHostAlloc) costs milliseconds and can serialise with
    the device, so the stream paths reuse theirs across calls (every call
    synchronises before returning, so reuse is safe)."""
    n = 1
    for d in shape:
        n *= int(d)
    buf = _pinned_cache.get((tag, dtype))
    if buf is None or buf.numel() < n:
        buf = torch.empty(max(n, 1), dtype=dtype, pin_memory=True)
        _pinned_cache[(tag, dtype)] = buf
    return buf[:n].view(*shape)


def stream_sweep(frames, stages, frac: float = 0.5, lap_scales=None, cap: int = 1 << 16,
                 d2h_cap: int = 4096):
    """A frame stream through the scale sweep (detect_sweep per frame) with
    the uploads overlapped: frame i+1's host-to-device copy runs on a copy
    stream while frame i's scales are filtered.  Every frame's results leave
    the device as soon as they exist (one asynchronous copy into pinned host
    memory per frame: counts, thresholds and the first d2h_cap detections
    of each scale; larger sets are completed at the end).  frames: (n, h, w)
    host array/tensor or a sequence of 2-D host tensors of one shape/dtype
    (pinned for full speed).  Returns per frame a list of Detections, one per
    stage."""
    if isinstance(frames, np.ndarray):
        frames = torch.from_numpy(np.ascontiguousarray(frames))
    frames = list(frames) if not isinstance(frames, torch.Tensor) else list(frames.unbind(0))
    if not frames or frames[0].ndim != 2:
        raise ValueError("frames must be a non-empty sequence of 2-D frames")
    dt = frames[0].dtype
    if dt not in (torch.uint16, torch.uint8, torch.float32):
        frames = [f.to(torch.float32) for f in frames]
        dt = torch.float32
    h, w = frames[0].shape
    code = {torch.uint16: _lib.VMF_U16, torch.uint8: _lib.VMF_U8}.get(dt, _lib.VMF_F32)
    stg = [s if isinstance(s, _Stage) else _Stage(s) for s in stages]
    ns, n = len(stg), len(frames)
    if ns == 0:
        return [[] for _ in frames]
    dev = torch.device("cuda", torch.cuda.current_device())
    cap = max(int(cap), 1)
    dcap = max(1, min(int(d2h_cap), cap))
    det_yx = torch.empty((n, ns, cap, 2), dtype=torch.int32, device=dev)
    det_val = torch.empty((n, ns, cap), dtype=torch.float32, device=dev)
    scal = torch.empty((n, ns, 2), dtype=torch.int64, device=dev)
    h_scal = _pinned("scal", (n, ns, 2), torch.int64)
    h_yx = _pinned("yx", (n, ns, dcap, 2), torch.int32)
    h_val = _pinned("val", (n, ns, dcap), torch.float32)
    up = _Uploader((h, w), dt)
    for i, f in enumerate(frames):
        if f.shape != (h, w) or f.dtype != dt:
            raise ValueError("all frames need one shape and dtype")
        x = up.put(f) if not f.is_cuda else f
        _sweep_launch(x, code, stg, frac, lap_scales, cap,
                      [(det_yx[i, j], det_val[i, j], scal[i, j]) for j in range(ns)])
        h_scal[i].copy_(scal[i], non_blocking=True)
        if os.environ.get("VMF_STREAM_PER_SCALE_D2H"):  # A/B: one copy per scale
            for j in range(ns):
                h_yx[i, j].copy_(det_yx[i, j, :dcap], non_blocking=True)
                h_val[i, j].copy_(det_val[i, j, :dcap], non_blocking=True)
        else:  # all scales in one strided copy each (fewer host-side calls per frame)
            h_yx[i].copy_(det_yx[i, :, :dcap], non_blocking=True)
            h_val[i].copy_(det_val[i, :, :dcap], non_blocking=True)
        if not f.is_cuda:
            up.release()
    torch.cuda.current_stream().synchronize()
    counts = h_scal[:, :, 0].tolist()
    thr = h_scal[:, :, 1:2].contiguous().view(torch.float32)[..., 0].tolist()
    out = []
    for i in range(n):
        row = []
        for j in range(ns):
            c = int(counts[i][j])
            m = min(c, cap)
            if m <= dcap:
                yx, val = h_yx[i, j, :m].numpy(), h_val[i, j, :m].numpy()
            else:
                yx, val = det_yx[i, j, :m].cpu().numpy(), det_val[i, j, :m].cpu().numpy()
            row.append(Detections(yx[:, 0].copy(), yx[:, 1].copy(), val.copy(), float(thr[i][j]),
                                  c, c > cap))
        out.append(row)
    return out


def pgm_stream_detect(paths, stage, frac: float = 0.5, cap: int = 1 << 16,
                      reference_units: bool = True, depth: int = 3):
    """Config-4 front end from files: binary PGM frames
    (P5, 16-bit big-endian or 8-bit, all the same size) through the fused
    single-scale path.  A reader thread readinto()s the raw sample bytes of
    frame i+depth-1 into a ring of pinned staging buffers while frame i is
    uploaded and filtered; the byte swap / widening to fp32 happens in the
    row pass (VMF_U16BE / VMF_U8), so the host never touches a sample.
    reference_units: scale L by 1/maxval, i.e. the values the reference
    computes from read_pgm's [0, 1] image.  Returns a list of Detections."""
    from concurrent.futures import ThreadPoolExecutor

    from .pgmio import pgm_info, read_pgm_raw

    paths = list(paths)
    if not paths:
        return []
    info0 = pgm_info(paths[0])
    if not info0.binary:
        raise ValueError(f"{paths[0]}: pgm_stream_detect needs binary (P5) PGMs")
    h, w = info0.height, info0.width
    wide = info0.maxval > 255
    nbytes = info0.nbytes
    depth = max(int(depth), 2)
    ring = [_pinned(f"ring{k}", (nbytes,), torch.uint8) for k in range(depth)]
    ring_free = [torch.cuda.Event() for _ in range(depth)]
    for e in ring_free:
        e.record(torch.cuda.current_stream())

    def load(i):
        slot = i % depth
        ring_free[slot].synchronize()  # the upload that last used this slot is done
        _, info = read_pgm_raw(paths[i], out=ring[slot].numpy())
        if (info.height, info.width, info.maxval > 255) != (h, w, wide):
            raise ValueError(f"{paths[i]}: frame shape/depth differs from {paths[0]}")
        return info

    stg = stage if isinstance(stage, _Stage) else _Stage(stage)
    res = _StreamResults(len(paths), cap)
    code = _lib.VMF_U16BE if wide else _lib.VMF_U8
    up = _Uploader((h, w), torch.uint16 if wide else torch.uint8)
    with ThreadPoolExecutor(max_workers=1) as pool:
        futs = [pool.submit(load, i) for i in range(min(depth, len(paths)))]
        for i in range(len(paths)):
            info = futs[i].result()
            slot = i % depth
            host = ring[slot][:nbytes].view(torch.uint16 if wide else torch.uint8).view(h, w)
            dbuf = up.put(host, after_copy=ring_free[slot])
            if i + depth < len(paths):
                futs.append(pool.submit(load, i + depth))
            scale = 1.0 / info.maxval if reference_units else 1.0
            _fused(dbuf, code, stg, stg, scale, frac, None, None, res.cap, False, out=res.out(i))
            up.release()
    return res.collect()
