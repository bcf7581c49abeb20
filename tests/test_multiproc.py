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
