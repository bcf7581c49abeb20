#!/usr/bin/env python
"""bench.py -- north-star benchmark of the B200-native vmfilt hot path.

Workload (BASELINE.json configs[2], the 4096^2 case the north-star target is
stated on): one 4096x4096 fp32 frame (2000 Gaussian blobs, s log-uniform
[2,32], A uniform [0.5,1.5], N(0, 0.05^2) noise; seeded synthetic, see
paper_1912_07133_b200/synth.py).  One STEP = the repeated-pole IIR scale
sweep sigma in {2,4,8,16,32}: per scale the fused path blur(rows) ->
blur(cols) -> Laplacian -> threshold (0.5 max|L|) + 3x3 NMS, i.e. five
passes of the hot path over the frame.  metric = Mpixel/s per scale
(frame pixels x scales / time).  The FIR family of the same sweep is timed
separately and reported in `per_scale` (IIR vs FIR, BASELINE.json metric).

Timing: W untimed warm-up steps; then K steps, each preceded by an L2 flush
(a 256 MiB memset, outside the events) and bracketed by CUDA events on the
launch stream; barrier + synchronize on both sides; max over ranks.
`value` = frame pixels x scales x ranks / time (weak scaling: every rank
processes its own frame; no data-path collective).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

SIGMAS = [2.0, 4.0, 8.0, 16.0, 32.0]
IIR = ["rp2", "rp4", "rp8", "rp16", "rp32"]
FIR = ["g2_k8", "g4_k16", "g8_k32", "g16_k64", "g32_k128"]
METRIC = "Mpixel/s per scale (IIR vs FIR) and achieved HBM GB/s vs B200 peak, 1 GPU"
UNIT = "Mpixel/s"
FLUSH_BYTES = 256 << 20
# algorithmic bytes per pixel per launch: fp32 read + write
# (the sweep's row pass reads X once and writes V of every scale: 4 + 4 ns;
# its column apply reads V: 4 -- the detect step keeps L in the apply's tiles,
# L is written only when asked for; the column carry reads V: 4)
ALGO_BYTES_PER_PX = {
    "iir_apply": 8, "iir_carry": 4, "iir_rows_fused": 8, "iir_cols_fused": 8,
    "fir_rows": 8, "fir_cols": 8, "laplacian": 8, "nms_count": 4, "nms_write": 4,
    "absmax": 4, "sweep_rows": 4 + 4 * 5, "col_apply": 4, "col_carry": 4,
}
# per scale, SURVEY §8(d)'s unit of the fused path (read X, write V, read V,
# write L), in which BASELINE's target is stated (>= 60 % of HBM == 245k
# Mpixel/s per scale); the detect step moves 12 of them (L stays on chip)
PATH_BYTES_PER_PX = 16
PATH_MOVED_BYTES_PER_PX = 12
# fp32 FMAs per pixel per scale of the modal K = 3 recursions (SURVEY §8(d)
# restated for the Laplacian-first path): per pass, chunk / band carries
# 2 directions x K, walks 2 directions x 2K (state + output), combine 2
FMA_PER_PX_PASS = {3: 6 * 3 + 2}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--size", type=int, default=4096)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the config 4 / 5 lines")
    ap.add_argument("--plumbing-check", action="store_true",
                    help="CPU/gloo check of the rank launch + max-over-ranks reduction only")
    return ap.parse_args()


def self_launch(args) -> bool:
    """`bench.py --gpus N` outside torchrun (no WORLD_SIZE): re-exec under
    torch.distributed.run with N ranks on this node (127.0.0.1) and pass its
    output through.  Returns True when this process was only the launcher."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    r = subprocess.run(cmd)
    if r.returncode:
        sys.exit(r.returncode)
    return True


def peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# nvidia-smi clock sampling during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev_index: int):
        self.dev = dev_index
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20", "-i", str(self.dev)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        busy = [s for s in sm if s > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# distributed plumbing (one process per GPU; weak scaling, no data collective)
# ---------------------------------------------------------------------------
def dist_init(backend, expect=None):
    import torch.distributed as dist

    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if expect is not None and ws != expect and not (ws == 1 and expect <= 1):
        raise SystemExit(f"bench.py: --gpus {expect} but WORLD_SIZE={ws}")
    if ws > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend)
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, local, ws


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(v, ws, device):
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(v)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# CPU side: the oracle port (test infrastructure) as baseline / reference arm
# ---------------------------------------------------------------------------
DFMA_PEAK_T = 16.44  # T fp64 FMA/s: profiles/r1_pipes.txt (tools/microbench/pipes.cu on this pool)
N_SM = 148


FIRTC_MIN_TAPS = 33  # vmf_firtc.cuh kFirTcMinTaps: from here the FIR runs on the tensor cores


def compute_roofline(per_scale, sweep_value, sm_mhz):
    """The arithmetic rooflines.  IIR (fp32 modal path): algorithmic fp32
    FMAs (FMA_PER_PX_PASS, both passes) against 148 SMs x 128 FMA/clk at the
    sampled SM clock, per single scale and for the 5-scale sweep.  FIR: below
    FIRTC_MIN_TAPS one DFMA per tap per pass against the measured DFMA peak;
    from there the tensor-core path, whose MMA work per pixel and pass is
    3 (3xTF32) x 2 x KW (the 128 + 2k window rounded up to 32) FLOP, against
    the TF32 dense peak taken as half the measured bf16 peak."""
    f32 = N_SM * 128 * (sm_mhz or 1965.0) * 1e6 / 1e12
    fma = 2 * FMA_PER_PX_PASS[3]
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            tf32 = float(json.load(fh)["bf16_tflops"]) / 2
        tf32_src = "MEASURED_PEAKS.json bf16_tflops / 2"
    except Exception:
        tf32, tf32_src = 1100.0, "B200_PROFILING.md nominal TF32 dense"
    out = {"iir_fp32": {"peak_tfma_s": round(f32, 2), "fma_per_px_scale": fma,
                        "sweep": {"tfma_s": round(sweep_value * 1e6 * fma / 1e12, 2),
                                  "frac": round(sweep_value * 1e6 * fma / 1e12 / f32, 3)},
                        "per_scale": {}},
           "fir": {"fp64_peak_tfma_s": DFMA_PEAK_T, "fp64_peak_source": "profiles/r1_pipes.txt",
                   "tf32_peak_tflop_s": round(tf32, 1), "tf32_peak_source": tf32_src,
                   "per_scale": {}}}
    for sg, v in per_scale["iir"].items():
        a = v * 1e6 * fma / 1e12
        out["iir_fp32"]["per_scale"][sg] = {"tfma_s": round(a, 2), "frac": round(a / f32, 3)}
    for sg, v in per_scale["fir"].items():
        taps = 2 * int(4 * float(sg)) + 1  # gaussian_fir(sigma, 0, 4 sigma)
        if taps >= FIRTC_MIN_TAPS:
            kw = -(-(128 + taps - 1) // 32) * 32
            a = v * 1e6 * 2 * 3 * 2 * kw / 1e12
            out["fir"]["per_scale"][sg] = {"taps": taps, "path": "tensor cores (3xTF32)",
                                           "mma_tflop_s": round(a, 1), "frac": round(a / tf32, 3),
                                           "useful_tflop_s": round(v * 1e6 * 4 * taps / 1e12, 1)}
        else:
            a = v * 1e6 * 2 * taps / 1e12
            out["fir"]["per_scale"][sg] = {"taps": taps, "path": "fp64 CUDA cores",
                                           "tfma_s": round(a, 2), "frac": round(a / DFMA_PEAK_T, 3)}
    return out


def cpu_stage_times(frame, stage, threads):
    """One scale through the oracle port, its three stages timed apart
    (blur, Laplacian, NMS), with `threads` host threads."""
    from oracle import oracle as O

    O.set_threads(threads)
    t0 = time.perf_counter()
    B = O.blur(frame, stage)
    t1 = time.perf_counter()
    L = O.laplacian(B)
    t2 = time.perf_counter()
    O.detect3x3(L, 0.5)
    t3 = time.perf_counter()
    return {"blur_ms": round(1e3 * (t1 - t0), 1), "laplacian_ms": round(1e3 * (t2 - t1), 1),
            "nms_ms": round(1e3 * (t3 - t2), 1), "threads": threads}


REF_DIR = os.path.join(REPO, "baseline", "_ref")


def ref_engine():
    """The reference package itself (vmfilt, pip-installed into baseline/_ref
    from /root/reference/pkg; numba JIT cache under /tmp), or None when it is
    not importable on this box."""
    if not os.path.isdir(os.path.join(REF_DIR, "vmfilt")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/vmfilt_numba_cache")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        from vmfilt import design, engine, polyz  # noqa: F401
    except Exception:
        return None
    return engine, design, polyz


def ref_stage(mods, st):
    """Our catalog stage -> the reference's own coefficient carrier."""
    engine, design, polyz = mods
    if hasattr(st, "taps"):
        return design.FirKernel(tuple(st.taps), st.parity, st.d)
    return polyz.ThreePartIIR(tuple(st.b_plus), tuple(st.a_plus), st.b_zero, st.parity)


def ref_scale(mods, frame, rst, lap):
    """One scale through the reference's own numba path (SURVEY.md §8(d),
    BASELINE.md §2): blur = apply_cols(apply_rows(x)) (engine.py:161-174),
    L = conv_rows(B, bank[2]) + conv_cols(B, bank[2]) (engine.py:205-228),
    stage 4 = the restated threshold + 3x3 NMS (no reference function)."""
    from oracle import oracle as O

    engine = mods[0]
    t0 = time.perf_counter()
    B = engine.apply_cols(engine.apply_rows(frame, rst), rst)
    t1 = time.perf_counter()
    L = engine.conv_rows(B, lap) + engine.conv_cols(B, lap)
    t2 = time.perf_counter()
    O.detect3x3(L, 0.5)
    t3 = time.perf_counter()
    return t3 - t0, {"blur_ms": round(1e3 * (t1 - t0), 1),
                     "laplacian_ms": round(1e3 * (t2 - t1), 1),
                     "nms_ms": round(1e3 * (t3 - t2), 1)}


def workload_config(h, w, n_gpus):
    """The `config` dict of both arms (identical, so the driver can match them)."""
    return {"workload": f"config3 {h}x{w} fp32, repeated-pole IIR sweep sigma 2..32, "
                        "blur+Laplacian+3x3 NMS per scale",
            "frame": [h, w], "scales": len(IIR), "parallelism": f"replicas x{n_gpus}"}


DTYPE = "f32"  # the IIR sweep: fp32 I/O, fp32 modal recursion state


def run_reference(args):
    """The reference's own CPU implementation on this host's cores: the
    reference package's numba kernels (kind "reference") when baseline/_ref
    imports here, else the C restatement in oracle/ (kind "port").  One step
    = one scale of the sweep (sigma cycling 2..32) on the full 4096^2 frame:
    a bounded sample of the 5-scale workload, same metric (Mpixel/s per
    scale)."""
    rank, local, ws = dist_init("gloo")
    if rank != 0:
        return
    from paper_1912_07133_b200 import filters, synth

    frame = synth.config3_frame(args.size).astype(np.float64)
    cat = filters.catalog()
    stages = [cat[n] for n in IIR]
    mpx = frame.size / 1e6
    threads = os.cpu_count() or 1
    mods = ref_engine()
    if mods is not None:
        engine, design, _ = mods
        engine.set_threads(threads)
        threads = engine.max_threads()
        lap = design.fir_vm_bank(3)[2]  # design hoisted out of the timed region
        rst = [ref_stage(mods, st) for st in stages]

        def one(i):
            return ref_scale(mods, frame, rst[i % len(rst)], lap)[0]
        kind = "reference"
        what = ("the reference package's numba path (baseline/_ref vmfilt: engine.apply_rows/"
                "apply_cols + conv_rows/conv_cols Laplacian, engine.py:35-228) + the restated "
                "3x3 NMS")
    else:
        from oracle import oracle as O

        O.set_threads(threads)

        def one(i):
            t0 = time.perf_counter()
            O.pipeline(frame, stages[i % len(stages)], frac=0.5)
            return time.perf_counter() - t0
        kind = "port"
        what = "oracle/vmf_oracle.c restatement of engine.py:35-102 + stage 4"
    for i in range(max(args.warmup, 1)):  # numba JIT + caches
        one(i)
    t = sum(one(i) for i in range(args.steps))
    value = mpx * args.steps / t
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.size, args.size, args.gpus),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"one scale per step (sigma cycling 2..32) on the full "
                                   f"{args.size}^2 frame, {args.steps} steps: {what}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch

    rank, local, ws = dist_init("nccl", expect=args.gpus)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_1912_07133_b200 import _lib, detect, filters, synth

    cat = filters.catalog()
    frame = synth.config3_frame(args.size)
    h, w = frame.shape
    mpx = h * w / 1e6
    x = torch.from_numpy(frame).to(dev)
    iir = [detect.make_stage(cat[n]) for n in IIR]
    fir = [detect.make_stage(cat[n]) for n in FIR]
    flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def one_scale(stg, frac=0.5):
        # the detect path of one scale (blur_laplacian_detect's device part):
        # detections only, L is not asked for
        detect._fused(x, _lib.VMF_F32, stg, stg, 1.0, frac, None, None, 1 << 18, False)

    # detection buffers of every scale, allocated up front (nothing is
    # allocated on the side streams inside a graph capture)
    outs = [(torch.empty((1 << 18, 2), dtype=torch.int32, device=dev),
             torch.empty(1 << 18, dtype=torch.float32, device=dev),
             torch.empty(2, dtype=torch.int64, device=dev)) for _ in IIR]

    def step(stages, conc=None):
        # the product sweep (detect_sweep's device part): scales on
        # concurrent streams, L of every scale written to its workspace
        detect._sweep_launch(x, _lib.VMF_F32, stages, 0.5, None, 1 << 18, outs, conc=conc)

    def timed(fn, n, flush_between=True):
        evs = []
        for _ in range(n):
            if flush_between:
                flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            evs.append((a, b))
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in evs)

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        step(iir)
    torch.cuda.synchronize()
    # one step = one CUDA graph replay (the 5-scale sweep), so host-side
    # launch overhead stays out of the device timeline
    n0 = _lib.launch_count()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step(iir)
    launches_per_step = _lib.launch_count() - n0
    graph.replay()
    torch.cuda.synchronize()
    barrier(ws)
    torch.cuda.synchronize()
    ms = timed(graph.replay, args.steps)
    launches = launches_per_step * args.steps
    torch.cuda.synchronize()
    barrier(ws)
    ms = max_over_ranks(ms, ws, dev)
    ms_step = ms / args.steps
    value = mpx * len(iir) * ws * args.steps / (ms / 1e3)

    # per-scale IIR vs FIR (BASELINE metric): each scale captured as its own
    # CUDA graph (device time, no host launch overhead), L2 flushed, 5 reps
    per_scale = {"iir": {}, "fir": {}}
    for fam, stages in (("iir", iir), ("fir", fir)):
        for sg, stg in zip(SIGMAS, stages):
            one_scale(stg)
            torch.cuda.synchronize()
            g1 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g1):
                one_scale(stg)
            g1.replay()
            torch.cuda.synchronize()
            t = timed(g1.replay, 5) / 5
            per_scale[fam][f"{sg:g}"] = round(mpx / (t / 1e3), 1)
            del g1

    # the finaliser at a low threshold (frac = 0.05: tens of thousands of
    # detections through the multi-CTA large-list path) against frac = 0.5,
    # one sigma = 4 scale each as its own graph
    low_frac = {}
    for fr in (0.5, 0.05):
        stg = iir[IIR.index("rp4")]
        one_scale(stg, fr)
        torch.cuda.synchronize()
        g1 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g1):
            one_scale(stg, fr)
        g1.replay()
        torch.cuda.synchronize()
        low_frac[f"frac_{fr:g}_ms"] = round(timed(g1.replay, 5) / 5, 4)
        del g1
    low_frac["ratio"] = round(low_frac["frac_0.05_ms"] / low_frac["frac_0.5_ms"], 3)

    # in-situ kernel timing over the same timed steps (events per launch)
    # (a second graph of the same step with event record nodes around every
    # launch: device-side durations without host launch gaps)
    # (the scales serialised on one stream here, so every launch's events
    # time that kernel alone; the headline step runs them concurrently)
    _lib.profile_begin()
    pgraph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(pgraph):
        step(iir, conc=1)
    _lib.profile_stop()
    prof = {}
    for _ in range(args.steps):
        flush.zero_()
        pgraph.replay()
        torch.cuda.synchronize()
        for k, (t, c) in _lib.profile_read().items():
            t0, c0 = prof.get(k, (0.0, 0))
            prof[k] = (t0 + t, c0 + c)
    clk = clocks.stop()
    hbm, peak_kind = peaks()
    dom = max(prof.items(), key=lambda kv: kv[1][0])
    dom_name, (dom_ms, dom_n) = dom
    per_launch_ms = dom_ms / dom_n
    algo = ALGO_BYTES_PER_PX.get(dom_name, 8) * h * w  # (sweep_rows: 5 scales per launch)
    achieved = algo / (per_launch_ms / 1e3) / 1e9
    traffic = None
    try:
        with open(os.path.join(REPO, "profiles", "ncu_traffic.json")) as fh:
            traffic = json.load(fh).get(dom_name)
    except Exception:
        pass
    path_gbs = PATH_BYTES_PER_PX * h * w * len(iir) / (ms_step / 1e3) / 1e9

    # end to end through the public API: K frames streamed from pinned host
    # memory through the 5-scale sweep (detect.stream_sweep): every step's
    # 64 MiB upload and its detections' readback are inside the timed
    # region; uploads overlap the previous frame's filtering.
    host = torch.from_numpy(frame).pin_memory()
    stages_obj = [cat[n] for n in IIR]
    # untimed pass of the same length: readback buffers allocated, PCIe link up to speed
    # at least 64 frames: a ~26 ms stream of 20 frames varied by +-15 % run to
    # run on one box (host-side jitter of the per-frame launch loop)
    ne2e = max(args.steps, 64)
    detect.stream_sweep([host] * ne2e, stages_obj)
    torch.cuda.synchronize()
    # median of 3 timed streams (a single 64-frame stream varied by ~4 % run
    # to run on the host side)
    e2e_runs = []
    for _ in range(3):
        barrier(ws)
        t0 = time.perf_counter()
        res = detect.stream_sweep([host] * ne2e, stages_obj)
        torch.cuda.synchronize()
        e2e_runs.append(max_over_ranks(time.perf_counter() - t0, ws, dev))
        assert len(res) == ne2e
    barrier(ws)
    e2e_s = sorted(e2e_runs)[1]
    d2h = len(iir) * (16 + 12 * 4096)  # per frame: header + first 4096 detections per scale
    e2e = mpx * len(iir) * ws * ne2e / e2e_s
    # the same without overlap: one detect_sweep call per frame (upload,
    # 5 scales, readback, then the next frame)
    detect.detect_sweep(host, stages_obj)
    torch.cuda.synchronize()
    barrier(ws)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        detect.detect_sweep(host, stages_obj)
    torch.cuda.synchronize()
    e2e1_s = max_over_ranks(time.perf_counter() - t0, ws, dev)
    barrier(ws)
    e2e_single = mpx * len(iir) * ws * args.steps / e2e1_s
    # the link the end-to-end number rides on: raw pinned H2D copies of one
    # frame (device-timed), and the Mpixel/s per scale they alone would allow
    dbuf = torch.empty_like(x)
    dbuf.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    ha, hb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ha.record(stream)
    for _ in range(5):
        dbuf.copy_(host, non_blocking=True)
    hb.record(stream)
    torch.cuda.synchronize()
    h2d_gbs = 5 * host.numel() * 4 / (ha.elapsed_time(hb) / 1e3) / 1e9
    del dbuf

    other = None
    if rank == 0 and ws == 1 and not args.no_extra:
        other = other_configs(cat, flush, stream)

    # parity of the benchmarked path at its own size: the sigma=4 scale of the
    # timed graph's last replay (detections) and of one more launch of the
    # same sweep with L written out, against the oracle on the same frame
    parity = None
    if rank == 0 and not args.no_cpu_baseline:
        graph.replay()  # outs <- the timed graph's detections
        torch.cuda.synchronize()
        parity = bench_parity(frame, cat, x, iir, outs)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_rows(frame, cat)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": DTYPE,
            "data": "synthetic",
            "config": workload_config(h, w, ws),
            "l2": "flushed (256 MiB memset) before every timed step",
            "parity": parity,
            "per_scale": per_scale,
            "low_threshold": dict(low_frac, scale="rp4 (sigma 4), 4096^2",
                                  note="frac 0.05 sends >4096 detections through the "
                                       "multi-CTA finaliser (VERDICT r1 item 5)"),
            "roofline": {"bound": "hbm", "kernel": dom_name, "achieved": round(achieved, 1),
                         "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": round(achieved / hbm, 4), "traffic": traffic,
                         "algo_bytes_per_launch": algo, "avg_launch_ms": round(per_launch_ms, 5)},
            "path_roofline": {"bytes_per_px": PATH_BYTES_PER_PX, "achieved": round(path_gbs, 1),
                              "peak": hbm, "frac": round(path_gbs / hbm, 4), "unit": "GB/s",
                              "note": "SURVEY 8(d) unit (16 B/px per scale; 60 % of HBM == "
                                      "245k Mpixel/s per scale); the detect step moves "
                                      f"{PATH_MOVED_BYTES_PER_PX} B/px (L stays in the column "
                                      "pass's tiles)",
                              "moved_frac": round(path_gbs * PATH_MOVED_BYTES_PER_PX
                                                  / PATH_BYTES_PER_PX / hbm, 4)},
            "compute_roofline": compute_roofline(per_scale, value / ws, clk.get("sm_mhz")),
            "kernels": {k: {"avg_ms": round(v[0] / v[1], 5), "launches": v[1]}
                        for k, v in prof.items()},
            "e2e": {"value": round(e2e, 1), "unit": UNIT,
                    "h2d_bytes_per_step": int(frame.nbytes),
                    "d2h_bytes_per_step": int(d2h),
                    "api": "detect.stream_sweep over K pinned frames (uploads overlapped)",
                    "frames": ne2e, "timed_streams": "median of 3",
                    "single_frame_value": round(e2e_single, 1),
                    "single_frame_api": "detect.detect_sweep per frame (no overlap)",
                    "h2d_gbs": round(h2d_gbs, 1),
                    "h2d_bound_value": round(h2d_gbs * 1e9 / frame.itemsize * len(iir) / 1e6, 1),
                    "h2d_note": "raw pinned H2D copy rate of one frame on this box, and the "
                                "Mpixel/s per scale that upload rate alone allows"},
            "gpu_launches": int(launches),
            "graph": "each timed step is one CUDA-graph replay of the 5-scale sweep "
                     f"(row pass for all scales, then each scale's column pass on its own stream); "
                     "`kernels` and `roofline` come from a serialised replay",
            "clocks": clk,
            "cpu_baseline": cpu,
            "other_configs": other,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def bench_parity(frame, cat, x, iir, outs):
    """Per-scale parity of the benchmarked sweep at 4096^2 (sigma = 4):
    L within 1e-4 max|L_ref|, blob set equal up to near-ties (tests/parity.py
    rule), against the oracle restatement on the same frame."""
    import torch

    from oracle import oracle as O
    from paper_1912_07133_b200 import _lib, detect
    from tests.parity import compare_blobs

    i = IIR.index("rp4")
    h, w = frame.shape
    cnt = int(outs[i][2][0].item())
    yx = outs[i][0][:cnt].cpu().numpy()
    got = set(zip(yx[:, 0].tolist(), yx[:, 1].tolist()))
    laps = [torch.empty((h, w), dtype=torch.float32, device=x.device) for _ in iir]
    extra = [(torch.empty_like(o[0]), torch.empty_like(o[1]), torch.empty_like(o[2])) for o in outs]
    detect._sweep_launch(x, _lib.VMF_F32, iir, 0.5, None, outs[0][1].numel(), extra, laps=laps)
    torch.cuda.synchronize()
    O.set_threads(os.cpu_count() or 1)
    B, L, (ys, xs, vs, thr) = O.pipeline(frame, cat["rp4"], frac=0.5)
    err = float(np.abs(laps[i].cpu().numpy().astype(np.float64) - L).max() / np.abs(L).max())
    want = set(zip(ys.tolist(), xs.tolist()))
    exempt, bad = compare_blobs(got, want, L, thr)
    return {"scale": "rp4 (sigma 4)", "lap_rel_err": err, "tol": 1e-4,
            "blob_set_equal": got == want, "blob_set_equal_up_to_near_ties": not bad,
            "n_blobs_gpu": len(got), "n_blobs_ref": len(want), "n_exempt": exempt,
            "oracle": "oracle/vmf_oracle.c (bit-identical to the reference's numba kernels on "
                      "tests/golden)"}


def cpu_baseline_rows(frame, cat):
    """cpu_baseline: the reference's own numba path on one sigma=4 scale of
    the same frame with all host threads (kind "reference"; falls back to
    the C port when baseline/_ref does not import), plus its 1-thread time
    and the C oracle port for comparison."""
    from oracle import oracle as O

    h, w = frame.shape
    mpx = h * w / 1e6
    threads = os.cpu_count() or 1
    f64 = frame.astype(np.float64)
    rows = {}
    O.set_threads(threads)
    O.pipeline(f64[:256, :256], cat["rp4"])
    pt = []
    for _ in range(3):
        t0 = time.perf_counter()
        O.pipeline(f64, cat["rp4"], frac=0.5)
        pt.append(time.perf_counter() - t0)
    port = {"value": round(mpx / statistics.median(pt), 2), "unit": UNIT, "cores": threads,
            "kind": "port", "sample": "median of 3, full frame, sigma 4 (oracle/vmf_oracle.c)",
            "stages": cpu_stage_times(f64, cat["rp4"], threads)}
    mods = ref_engine()
    if mods is None:
        port["reference_unavailable"] = "baseline/_ref (vmfilt + numba) does not import here"
        return port
    engine, design, _ = mods
    lap = design.fir_vm_bank(3)[2]
    rst = ref_stage(mods, cat["rp4"])
    for nthr in (threads, 1):
        engine.set_threads(nthr)
        ref_scale(mods, f64[:512, :512], rst, lap)  # JIT
        ts, st = [], None
        for _ in range(3 if nthr > 1 else 1):
            t, st = ref_scale(mods, f64, rst, lap)
            ts.append(t)
        rows[nthr] = (statistics.median(ts), st, engine.max_threads())
    t, st, used = rows[threads]
    return {"value": round(mpx / t, 2), "unit": UNIT, "cores": used, "kind": "reference",
            "sample": f"full {h}x{w} frame, sigma=4 repeated-pole scale, median of 3: the "
                      "reference package's numba path (baseline/_ref vmfilt engine.apply_rows/"
                      "apply_cols, conv_rows/conv_cols Laplacian) + the restated 3x3 NMS",
            "stages": st,
            "one_thread": {"value": round(mpx / rows[1][0], 2), "stages": rows[1][1]},
            "port": port}


def other_configs(cat, flush, stream):
    """Secondary lines (rank 0, N=1): config 4 (u16 stream, sustained end to
    end with double-buffered uploads) and config 5 (8192^2, Butterworth IIR vs
    385-tap SG FIR per scale).  Device-timed values are CUDA-graph replays
    with L2 flushed before each rep."""
    import torch

    from paper_1912_07133_b200 import _lib, detect, synth

    out = {}

    def graph_ms(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        g.replay()
        torch.cuda.synchronize()
        tot = 0.0
        for _ in range(reps):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g.replay()
            b.record(stream)
            b.synchronize()
            tot += a.elapsed_time(b)
        del g
        return tot / reps

    # config 4: the config's 64-frame stream of 2048^2 u16, rp6, per-frame
    # threshold + NMS
    frames = synth.config4_stream(n_frames=64)
    n4, h4, w4 = frames.shape
    host = torch.from_numpy(frames).pin_memory()
    st4 = detect.make_stage(cat["rp6"])
    detect.stream_detect(host, st4)  # untimed pass of the same length (PCIe link, buffers)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = detect.stream_detect(host, st4)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    dframes = host.cuda()
    x4 = dframes[0]
    lap4 = torch.empty((h4, w4), dtype=torch.float32, device=x4.device)
    ms4 = graph_ms(lambda: detect._fused(x4, _lib.VMF_U16, st4, st4, 1.0, 0.5, None, lap4,
                                         1 << 16, False))
    mpx4 = h4 * w4 / 1e6
    # the same 16 frames device-resident, 3 in flight (one CUDA graph)
    outs4 = [(torch.empty((1 << 16, 2), dtype=torch.int32, device=x4.device),
              torch.empty(1 << 16, dtype=torch.float32, device=x4.device),
              torch.empty(2, dtype=torch.int64, device=x4.device)) for _ in range(n4)]
    ms4s = graph_ms(lambda: detect._sweep_launch([dframes[i] for i in range(n4)], _lib.VMF_U16,
                                                 [st4] * n4, 0.5, None, 1 << 16, outs4))
    out["config4"] = {
        "workload": f"{n4} frames {h4}x{w4} u16, rp6 blur + Laplacian + 3x3 NMS per frame",
        "e2e_sustained_mpx_s": round(mpx4 * n4 / e2e_s, 1),
        "e2e_note": "pinned host frames -> device (copy stream, 2 buffers) -> detections back",
        "device_mpx_s": round(mpx4 / (ms4 / 1e3), 1),
        "device_stream_mpx_s": round(mpx4 * n4 / (ms4s / 1e3), 1),
        "device_stream_note": f"{n4} device-resident frames, 3 in flight on concurrent streams "
                              "(stream_detect's device part), one CUDA graph",
        "detections_per_frame": int(statistics.median([r.count for r in res]))}
    del dframes, x4, lap4, outs4

    # config 3 with the scale-space rule: sigma^2-normalised L of the 5 IIR
    # scales into one stack, 3x3x3 NMS over it (detect.scale_space_detect's
    # device part; the per-scale passes on concurrent streams)

    f3 = synth.config3_frame(4096)
    x3 = torch.from_numpy(f3).cuda()
    sig3 = (2, 4, 8, 16, 32)
    st3 = [detect.make_stage(cat[f"rp{s}"]) for s in sig3]
    stack = torch.empty((5, 4096, 4096), dtype=torch.float32, device=x3.device)
    cands3 = (torch.empty((5, detect.SS_CAND_CAP, 2), dtype=torch.int32, device=x3.device),
              torch.empty((5, detect.SS_CAND_CAP), dtype=torch.float32, device=x3.device),
              torch.empty((5, 2), dtype=torch.int64, device=x3.device))
    det3 = torch.empty((1 << 18, 3), dtype=torch.int32, device=x3.device)
    val3 = torch.empty(1 << 18, dtype=torch.float32, device=x3.device)
    scal3 = torch.zeros(2, dtype=torch.int64, device=x3.device)

    def ss_step():  # the stack planes + per-scale candidates, then the 3x3x3 rule on them
        detect._scale_space_launch(x3, _lib.VMF_F32, st3, sig3, 0.5, stack, cands3, det3, val3,
                                   scal3)

    ms3 = graph_ms(ss_step)
    assert int(scal3[0].item()) >= 0, "a scale's candidate list overflowed"
    out["config3_scale_space"] = {
        "workload": "4096x4096 fp32, 5 repeated-pole scales, sigma^2-normalised L stack, "
                    "3x3x3 NMS at 0.5 max|stack|",
        "mpx_s_per_scale": round(5 * 4096 * 4096 / 1e6 / (ms3 / 1e3), 1),
        "ms_per_sweep": round(ms3, 4)}
    del x3, stack, cands3

    # config 5: 8192^2 fp32, Butterworth sigma 48 (K=2) vs colored SG 385 taps
    f5 = synth.config5_frame(8192)
    x5 = torch.from_numpy(f5).cuda()
    c5 = {"workload": "8192x8192 fp32, bw48 IIR vs sg38.4 (385-tap) FIR, fused blur + "
                      "Laplacian + 3x3 NMS"}
    for name in ("bw48", "sg38.4"):
        stg = detect.make_stage(cat[name])
        ms = graph_ms(lambda: detect._fused(x5, _lib.VMF_F32, stg, stg, 1.0, 0.5, None, None,
                                            1 << 18, False))
        c5[name + "_mpx_s"] = round(8192 * 8192 / 1e6 / (ms / 1e3), 1)
    out["config5"] = c5
    del x5
    return out


def plumbing_check(args):
    """The multi-rank plumbing of run_ours without a GPU: gloo process group,
    barrier, max over ranks of a rank-dependent value, world == --gpus."""
    rank, local, ws = dist_init("gloo", expect=args.gpus)
    barrier(ws)
    v = max_over_ranks(float(rank + 1), ws, "cpu")
    barrier(ws)
    if rank == 0:
        print(json.dumps({"n_gpus": ws, "max_over_ranks": v}), flush=True)
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def main():
    args = parse()
    if self_launch(args):
        return
    if args.plumbing_check:
        plumbing_check(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
