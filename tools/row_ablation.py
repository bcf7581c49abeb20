"""Timing ablations of the sweep row pass (results of the ablated builds are
invalid; only their kernel times are read).  Builds: build/abl/libablN.so
with -DVMF_ABL=N (1: no chunk scans, 2: no walks, 3: no carries).
python tools/row_ablation.py -> one JSON line per build: sweep_rows us, step ms."""
import json
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--one":
    sys.path.insert(0, ".")
    import torch
    from paper_1912_07133_b200 import _lib, detect, filters, synth

    cat = filters.catalog()
    x = torch.from_numpy(synth.config3_frame(4096)).cuda()
    stg = [detect.make_stage(cat[n]) for n in ["rp2", "rp4", "rp8", "rp16", "rp32"]]
    outs = [(torch.empty((1 << 18, 2), dtype=torch.int32, device="cuda"),
             torch.empty(1 << 18, dtype=torch.float32, device="cuda"),
             torch.empty(2, dtype=torch.int64, device="cuda")) for _ in stg]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    step = lambda conc: detect._sweep_launch(x, _lib.VMF_F32, stg, 0.5, None, 1 << 18, outs, conc=conc)
    for _ in range(3):
        step(3)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step(3)
    tot = 0.0
    for _ in range(20):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); b.synchronize()
        tot += a.elapsed_time(b)
    _lib.profile_begin()
    pg = torch.cuda.CUDAGraph()
    with torch.cuda.graph(pg):
        step(1)
    _lib.profile_stop()
    prof = {}
    for _ in range(10):
        flush.zero_()
        pg.replay(); torch.cuda.synchronize()
        for k, (t, c) in _lib.profile_read().items():
            t0, c0 = prof.get(k, (0.0, 0)); prof[k] = (t0 + t, c0 + c)
    print(json.dumps({"lib": os.environ.get("VMF_LIB_PATH", "main"), "step_ms": round(tot / 20, 4),
                      "kernels_us": {k: round(1e3 * t / c, 2) for k, (t, c) in prof.items()}}))
    sys.exit(0)

libs = [None] + sorted(os.path.join("build/abl", f) for f in os.listdir("build/abl") if f.endswith(".so"))
for lib in libs:
    env = dict(os.environ)
    if lib:
        env["VMF_LIB_PATH"] = os.path.abspath(lib)
    r = subprocess.run([sys.executable, __file__, "--one"], env=env, capture_output=True, text=True)
    print(r.stdout.strip() or r.stderr[-800:], flush=True)
