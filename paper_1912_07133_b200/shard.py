"""Multi-GPU sharding of the hot path.

The path partitions into independent units -- frames of a stream (config 4)
or scales of a sweep (config 3) -- so N GPUs run N replicas with no
data-path collective: rank r takes units r, r + N, r + 2N, ...  The only
cross-rank traffic is the timing reduction (max over ranks) and gathering
per-unit detection counts, both plumbing done with torch.distributed.
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
