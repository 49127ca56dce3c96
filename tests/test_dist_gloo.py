"""Multi-process (world_size 2, gloo, CPU) checks of the multi-GPU host logic: head
sharding covers every head exactly once, max-over-ranks timing, and the verification
gathers -- the same functions bench.py uses over NCCL."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_12675_b200 import dist as sd


def test_head_range_partition():
    for H in (1, 2, 12, 40):
        for world in (1, 2, 4, 8):
            shards = sd.all_shards(H, world)
            covered = [h for a, b in shards for h in range(a, b)]
            assert covered == list(range(H))
            sizes = [b - a for a, b in shards]
            assert max(sizes) - min(sizes) <= 1
    assert sd.all_shards(40, 8) == [(5 * r, 5 * r + 5) for r in range(8)]
    assert [b - a for a, b in sd.all_shards(12, 8)] == [2, 2, 2, 2, 1, 1, 1, 1]
    with pytest.raises(ValueError):
        sd.head_range(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = sd.max_over_ranks(1.5 + rank)
        out = torch.full((2, 3), float(rank + 1))
        cs = sd.gather_checksums(out)
        outs = sd.gather_outputs(out)
        h0, h1 = sd.head_range(40, world, rank)
        q.put((rank, t, cs, [float(o.sum()) for o in outs], (h0, h1)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_timing_and_gather():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, t, cs, sums, shard in res:
        assert t == 2.5                      # max over ranks
        assert cs == [6.0, 12.0]             # rank r contributes 6 * (r + 1)
        assert sums == [6.0, 12.0]
    assert [r[4] for r in res] == [(0, 20), (20, 40)]
