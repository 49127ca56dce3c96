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


def _shard_worker(rank, world, port, q):
    """Uneven head shards (H = 5 over 2 ranks: 3 + 2): every rank's per-head tensors gathered in
    head order, sampled heads fetched from their owners."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        H = 5
        h0, h1 = sd.head_range(H, world, rank)
        local = torch.stack([torch.full((3, 4), float(h), dtype=torch.float32) for h in range(h0, h1)])
        masks = sd.gather_head_shards(local.to(torch.uint8), H, world, rank)
        sampled = sd.gather_sampled_heads(local, [0, 4], H, world, rank)
        q.put((rank, [int(masks[h, 0, 0]) for h in range(H)], {h: float(t[0, 0]) for h, t in sampled.items()}))
    finally:
        dist.destroy_process_group()


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


def test_gloo_world2_shard_gathers():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, masks, sampled in res:
        assert masks == [0, 1, 2, 3, 4]
        assert sampled == {0: 0.0, 4: 4.0}


def test_head_inputs_are_per_head():
    """A shard's inputs equal the heads generated one by one (any rank can regenerate any head)."""
    q, k, v, pq, pk, rho = sd.shard_inputs(1, 3, 1, 256, 128, 2, torch.float32, torch.device("cpu"))
    hq, hk, hv, hpq, hpk, hrho = sd.head_inputs(2, 256, 128, 2, torch.float32, torch.device("cpu"))
    assert torch.equal(q[0, 1], hq) and torch.equal(v[0, 1], hv) and torch.equal(pk[1], hpk) and torch.equal(rho[1], hrho)


def test_bench_gpus2_plumbing_verified():
    """`python bench.py --gpus 2` on a box without CUDA: it relaunches itself as 2 ranks (gloo),
    shards the heads, gathers every mask and two output heads to rank 0 and verifies them
    against the oracle (CPU stand-in compute: no value is reported)."""
    import json
    import subprocess
    import sys
    if torch.cuda.is_available():
        pytest.skip("GPU present: bench.py runs the CUDA path")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--config", "cfg2"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong" and line["value"] is None
    assert line["parity"]["pass"] and line["parity"]["mask_rows_mismatched"] == 0
    assert line["parity"]["heads_masks_checked"] == line["config"]["H"]
