"""shard.scale_space_detect over NCCL on two GPUs (one process each): the
halo planes travel by batched P2P, the maximum by all-reduce, and the union
of the ranks' detections equals the single-process scale-space detector.
Runs only where two GPUs are visible (the driver's round-end box has one;
test_multiproc.py covers the same host logic with gloo on CPU)."""
import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu

needs_two = pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                               reason="needs two GPUs")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, subgroup, q):
    import torch.distributed as dist

    from paper_1912_07133_b200 import filters, shard, synth

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    group = dist.new_group(list(range(world))) if subgroup else None
    cat = filters.catalog()
    spec = synth.CONFIG_STAGES[3]
    x = torch.from_numpy(synth.config3_frame(1024)).cuda()
    d = shard.scale_space_detect(x, [cat[n] for n in spec["iir"]], spec["sigmas"], frac=0.5,
                                 group=group)
    q.put((rank, d.threshold, sorted(zip(d.s.tolist(), d.y.tolist(), d.x.tolist()))))
    dist.barrier()
    dist.destroy_process_group()


@needs_two
@pytest.mark.parametrize("subgroup", [False, True])
def test_scale_sharded_detect_nccl_world2(cat, subgroup):
    import torch.multiprocessing as mp

    from paper_1912_07133_b200 import detect, synth

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, subgroup, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    spec = synth.CONFIG_STAGES[3]
    ref = detect.scale_space_detect(synth.config3_frame(1024), [cat[n] for n in spec["iir"]],
                                    spec["sigmas"], frac=0.5)
    got = sorted(t for _, _, dets in res for t in dets)
    want = sorted(zip(ref.s.tolist(), ref.y.tolist(), ref.x.tolist()))
    assert all(thr == ref.threshold for _, thr, _ in res)
    assert got == want
