"""Multi-GPU sharding of the hot path.

The path partitions into independent units -- frames of a stream (config 4)
or scales of a sweep (config 3) -- so N GPUs run N replicas with no
data-path collective: rank r takes units r, r + N, r + 2N, ...  The only
cross-rank traffic is the timing reduction (max over ranks) and gathering
per-unit detection counts, both plumbing done with torch.distributed.

The scale-space rule of config 3 (3x3x3 NMS over the sigma^2-normalised
stack at 0.5 max|stack|) is the one exchange step the path has:
scale_space_detect gives each rank a contiguous block of scales, then
exchanges one L map each way with its neighbours (point-to-point, NCCL over
NVLink on GPUs) and all-reduces the stack maximum, so every rank's NMS sees
exactly the neighbours and threshold of the unsharded stack.
"""
from __future__ import annotations


def units_for_rank(n_units: int, rank: int, world: int) -> list:
    """Round-robin assignment; every unit exactly once across ranks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return list(range(rank, n_units, world))


def detect_stream(frames, stage, frac: float = 0.5, rank: int = 0, world: int = 1,
                  cap: int = 1 << 18):
    """Config-4 stream: fused blur + Laplacian + NMS on this rank's frames.

    frames: (n, h, w) array (uint16 or float32), host or device.  Returns
    {frame index: Detections} for the frames this rank owns."""
    from .detect import blur_laplacian_detect

    out = {}
    for i in units_for_rank(len(frames), rank, world):
        out[i] = blur_laplacian_detect(frames[i], stage, frac=frac, cap=cap)
    return out


def scale_blocks(n_units: int, world: int) -> list:
    """Contiguous blocks [lo, hi) per rank, sizes differing by at most one
    (ranks beyond n_units get empty blocks at the end)."""
    if world < 1:
        raise ValueError("bad world size")
    base, extra = divmod(n_units, world)
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def exchange_halos(stack, has_lo: bool, has_hi: bool, rank: int, group=None) -> None:
    """stack = [halo_lo?] + own planes + [halo_hi?] (a 3-D tensor, own planes
    filled): send the first own plane down and the last one up, receive the
    neighbours' edge planes into the halo slots (batched P2P)."""
    import torch.distributed as dist

    def peer(r):  # P2POp takes a GLOBAL rank; `rank` is the rank within `group`
        return r if group is None else dist.get_global_rank(group, r)

    n = stack.shape[0]
    first, last = (1 if has_lo else 0), n - (2 if has_hi else 1)
    ops = []
    if has_lo:
        ops.append(dist.P2POp(dist.isend, stack[first].contiguous(), peer(rank - 1), group))
        ops.append(dist.P2POp(dist.irecv, stack[0], peer(rank - 1), group))
    if has_hi:
        ops.append(dist.P2POp(dist.isend, stack[last].contiguous(), peer(rank + 1), group))
        ops.append(dist.P2POp(dist.irecv, stack[n - 1], peer(rank + 1), group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def global_max(value, group=None):
    """All-reduce MAX of a one-element tensor (the stack maximum)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(value, op=dist.ReduceOp.MAX, group=group)
    return value


def own_detections(s, lo: int, has_lo: bool, n_own: int):
    """Mask of the detections on this rank's own planes and their global
    scale indices (local plane s -> lo + s - has_lo)."""
    import numpy as np

    s = np.asarray(s)
    keep = (s >= int(has_lo)) & (s < int(has_lo) + n_own)
    return keep, s[keep] - int(has_lo) + lo


def scale_space_detect(img, stages, sigmas, frac: float = 0.5, cap: int = 1 << 18,
                       group=None):
    """detect.scale_space_detect over the ranks of `group` (or one process):
    this rank computes the L maps of its scale block (sigma^2-normalised, the
    block's scales on concurrent streams), exchanges halo planes, all-reduces
    the maximum and runs the 3x3x3 NMS on its slab with that threshold.
    Returns this rank's Detections (s = global scale index)."""
    import ctypes as C

    import numpy as np
    import torch
    import torch.distributed as dist

    from . import _lib
    from .detect import Detections, _Stage, _sweep_launch
    from .engine import _as_image, _ptr, _stream, _workspace

    if len(stages) != len(sigmas) or not stages:
        raise ValueError("need one stage per sigma")
    dist_on = dist.is_available() and dist.is_initialized()
    rank = dist.get_rank(group) if dist_on else 0
    world = dist.get_world_size(group) if dist_on else 1
    ns = len(stages)
    lo, hi = scale_blocks(ns, world)[rank]
    n_own = hi - lo
    has_lo, has_hi = n_own > 0 and lo > 0, n_own > 0 and hi < ns
    x, kind, code = _as_image(img)
    h, w = x.shape
    dev = x.device
    stack = torch.zeros((max(n_own, 0) + has_lo + has_hi or 1, h, w), dtype=torch.float32,
                        device=dev)
    if n_own:
        own = [stack[int(has_lo) + i] for i in range(n_own)]
        dummy = [(torch.empty((1, 2), dtype=torch.int32, device=dev),
                  torch.empty(1, dtype=torch.float32, device=dev),
                  torch.empty(2, dtype=torch.int64, device=dev)) for _ in range(n_own)]
        _sweep_launch(x, code, [_Stage(st) for st in stages[lo:hi]], 0.0,
                      [float(sg) ** 2 for sg in sigmas[lo:hi]], 0, dummy, laps=own)
        mx = stack[int(has_lo):int(has_lo) + n_own].abs().amax().reshape(1)
    else:
        mx = torch.zeros(1, dtype=torch.float32, device=dev)
    if world > 1:
        # every rank of the group takes part in the all-reduce first, so the
        # batched P2P below is never the group's first collective (NCCL needs
        # all ranks in that one; ranks without scales send nothing)
        global_max(mx, group)
        exchange_halos(stack, has_lo, has_hi, rank, group)
    if not n_own:
        return Detections(np.empty(0, np.int32), np.empty(0, np.int32),
                          np.empty(0, np.float32), float(frac * mx.item()), 0, False,
                          s=np.empty(0, np.int32))
    L = _lib.lib()
    nsl = stack.shape[0]
    ws = _workspace(L.vmf_detect3x3x3_workspace_bytes(nsl, h, w))
    cap = max(int(cap), 1)
    # the slab's list also holds the halo planes' detections (sorted first for
    # the lower halo), so its capacity covers them; a slab list that still
    # overflows is redone at its exact size, so the own-plane count is exact
    slab_cap = cap * (1 + int(has_lo) + int(has_hi))
    while True:
        det = torch.empty((slab_cap, 3), dtype=torch.int32, device=dev)
        val = torch.empty((slab_cap,), dtype=torch.float32, device=dev)
        scal = torch.zeros(2, dtype=torch.int64, device=dev)
        n_host = C.c_int64(0)
        _lib.check(L.vmf_detect3x3x3_absmax(
            _ptr(stack), nsl, h, w, w, h * w, float(frac), _ptr(mx), _ptr(det), _ptr(val),
            slab_cap, _ptr(scal), scal.data_ptr() + 8, C.byref(n_host), _ptr(ws), ws.numel(),
            _stream()))
        n = n_host.value
        if n <= slab_cap:
            break
        slab_cap = n
    thr = float(scal[1:2].view(torch.float32)[0].item())
    d, v = det[:n].cpu().numpy(), val[:n].cpu().numpy()
    keep, s_glob = own_detections(d[:, 0], lo, has_lo, n_own)
    n_mine = int(keep.sum())
    ys, xs, vs, ss = d[keep, 1][:cap], d[keep, 2][:cap], v[keep][:cap], s_glob[:cap]
    return Detections(ys, xs, vs, thr, n_mine, n_mine > cap, s=ss.astype(np.int32))
