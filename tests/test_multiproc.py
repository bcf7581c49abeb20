"""World-size-2 gloo checks of the multi-GPU plumbing on CPU: the unit
sharding covers every frame exactly once and the max-over-ranks timing
reduction used by bench.py is correct."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1912_07133_b200.shard import units_for_rank


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_units, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = units_for_rank(n_units, rank, world)
    # gather every rank's units (what a rank-0 report would do)
    lists = [None] * world
    dist.all_gather_object(lists, mine)
    # bench.py's reduction: max over ranks of the per-rank device time
    t = torch.tensor([float(rank + 1) * 1.5], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.barrier()
    q.put((rank, lists, float(t.item())))
    dist.destroy_process_group()


@pytest.mark.parametrize("n_units", [64, 5, 1])
def test_sharding_and_max_reduction_world2(n_units):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_units, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, lists, tmax in res:
        flat = sorted(u for lst in lists for u in lst)
        assert flat == list(range(n_units))  # every unit exactly once
        assert tmax == 3.0                   # max over ranks, not rank-local


def test_units_for_rank_validation():
    assert units_for_rank(10, 1, 3) == [1, 4, 7]
    with pytest.raises(ValueError):
        units_for_rank(10, 3, 3)


def _ss_worker(rank, world, port, q, sub=None):
    """The scale-sharded 3x3x3 NMS host logic on CPU (gloo): block partition,
    halo exchange, all-reduced maximum, own-plane filtering -- with the
    oracle's NMS standing in for the device kernel."""
    import numpy as np

    from oracle import oracle as O
    from paper_1912_07133_b200 import shard

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    group = None
    if sub is not None:  # a non-default group: P2P peers are group ranks -> global ranks
        group = dist.new_group(sub)
        if rank not in sub:
            q.put((rank, None, None))
            dist.destroy_process_group()
            return
        rank, world = dist.get_rank(group), len(sub)
    full = np.random.default_rng(5).standard_normal((5, 24, 20)).astype(np.float32)
    full[2, 10, 10] = 9.0          # a strong extremum in the middle scale
    full[0, 5, 5] = -8.0           # and on the first scale (one-sided in s)
    lo, hi = shard.scale_blocks(5, world)[rank]
    n_own = hi - lo
    has_lo, has_hi = n_own > 0 and lo > 0, n_own > 0 and hi < 5
    slab = torch.zeros((n_own + has_lo + has_hi or 1, 24, 20), dtype=torch.float32)
    if n_own:
        slab[int(has_lo):int(has_lo) + n_own] = torch.from_numpy(full[lo:hi])
        mx = slab[int(has_lo):int(has_lo) + n_own].abs().amax().reshape(1)
    else:
        mx = torch.zeros(1)
    shard.global_max(mx, group)  # first: never a P2P batch as the group's first collective
    shard.exchange_halos(slab, has_lo, has_hi, rank, group)
    got = []
    if n_own:
        ss, ys, xs, vs, thr = O.detect3x3x3(slab.numpy(), thr=0.5 * float(mx.item()))
        keep, sg = shard.own_detections(ss, lo, has_lo, n_own)
        got = sorted(zip(sg.tolist(), ys[keep].tolist(), xs[keep].tolist()))
    allgot = [None] * world
    dist.all_gather_object(allgot, got, group=group)
    q.put((rank, allgot, float(mx.item())))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,sub", [(2, None), (3, None), (7, None), (4, (1, 2, 3))])
def test_scale_sharded_nms_equals_unsharded(world, sub):
    import numpy as np

    from oracle import oracle as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ss_worker, args=(r, world, port, q, sub)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = np.random.default_rng(5).standard_normal((5, 24, 20)).astype(np.float32)
    full[2, 10, 10] = 9.0
    full[0, 5, 5] = -8.0
    ss, ys, xs, vs, thr = O.detect3x3x3(full.astype(np.float64), frac=0.5)
    want = sorted(zip(ss.tolist(), ys.tolist(), xs.tolist()))
    assert len(want) >= 2
    res = [r for r in res if r[1] is not None]
    assert len(res) == (len(sub) if sub else world)
    for rank, allgot, mx in res:
        assert mx == pytest.approx(9.0)
        assert sorted(d for part in allgot for d in part) == want
