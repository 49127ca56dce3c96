"""Multi-GPU plumbing for the SLA2 forward (one process per GPU, torch.distributed).

SLA2's state is per (batch, head): the column mean, router projections, alpha logits, the
linear-branch totals and the kept-block lists all live inside one (b, h) slice
(model.hpp:38-39, attention.hpp:423-560), so the forward shards by head with no collective in
the data path. Collectives are used only for
  * timing: the max over ranks of each rank's device time (the job is as slow as its slowest
    rank), and
  * verification: an all-gather of per-rank output checksums (and optionally of outputs).
"""
from __future__ import annotations

from typing import List, Tuple


def head_range(H: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous head shard [h0, h1) of rank `rank`: sizes differ by at most one, larger
    shards first (H = 12 over 8 ranks -> 2,2,2,2,1,1,1,1; H = 40 over 8 -> 5 each)."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(H, world)
    h0 = rank * base + min(rank, extra)
    return h0, h0 + base + (1 if rank < extra else 0)


def all_shards(H: int, world: int) -> List[Tuple[int, int]]:
    return [head_range(H, world, r) for r in range(world)]


def max_over_ranks(value: float, device=None) -> float:
    """Max of a float across ranks (all_reduce MAX); identity without a process group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_checksums(out, device=None) -> List[float]:
    """All-gather a float64 checksum (sum) of each rank's output -- verification only."""
    import torch
    import torch.distributed as dist
    cs = out.double().sum().reshape(1).to(device if device is not None else out.device)
    if not (dist.is_available() and dist.is_initialized()):
        return [float(cs.item())]
    bufs = [torch.zeros_like(cs) for _ in range(dist.get_world_size())]
    dist.all_gather(bufs, cs)
    return [float(b.item()) for b in bufs]


def head_inputs(h: int, N: int, d: int, tm: int, dtype, device, seed_base: int = 1234):
    """Synthetic inputs of GLOBAL head h, a function of (seed_base + h) only, so that any rank
    can regenerate any head (rank 0 does, to verify the gathered shards): q, k, v [N, d] ~
    N(0, 1) in `dtype`; proj_q, proj_k = I + 0.05 N(0, 1) [d, d] (test_gradients.cpp:143-148);
    rho ~ U(-1, 1) [tm] (:149), fp32."""
    import torch
    g = torch.Generator(device=device).manual_seed(seed_base + h)
    q = torch.randn((N, d), generator=g, device=device).to(dtype)
    k = torch.randn((N, d), generator=g, device=device).to(dtype)
    v = torch.randn((N, d), generator=g, device=device).to(dtype)
    eye = torch.eye(d, device=device)
    pq = eye + 0.05 * torch.randn((d, d), generator=g, device=device)
    pk = eye + 0.05 * torch.randn((d, d), generator=g, device=device)
    rho = torch.rand((tm,), generator=g, device=device) * 2 - 1
    return q, k, v, pq.contiguous(), pk.contiguous(), rho.contiguous()


def shard_inputs(h0: int, h1: int, B: int, N: int, d: int, tm: int, dtype, device, seed_base: int = 1234):
    """The [h0, h1) head shard as forward() operands: q, k, v [B, h1-h0, N, d] (batch entry b of
    head h uses seed_base + b * 100003 + h), proj_q, proj_k [h1-h0, d, d], rho [h1-h0, tm]
    (per-head router state shared across the batch, model.hpp:38-39)."""
    import torch
    Hs = h1 - h0
    q = torch.empty((B, Hs, N, d), dtype=dtype, device=device)
    k, v = torch.empty_like(q), torch.empty_like(q)
    pq = torch.empty((Hs, d, d), dtype=torch.float32, device=device)
    pk, rho = torch.empty_like(pq), torch.empty((Hs, tm), dtype=torch.float32, device=device)
    for b in range(B):
        for j, h in enumerate(range(h0, h1)):
            hq, hk, hv, hpq, hpk, hrho = head_inputs(h, N, d, tm, dtype, device, seed_base + b * 100003)
            q[b, j], k[b, j], v[b, j] = hq, hk, hv
            if b == 0:
                pq[j], pk[j], rho[j] = hpq, hpk, hrho
    return q, k, v, pq, pk, rho


def gather_head_shards(local, H: int, world: int, rank: int):
    """All-gather per-head tensors sharded by head_range: `local` is [h1-h0, ...] on every rank;
    returns [H, ...] (every rank) -- masks / index lists for verification, untimed. Shards are
    padded to the largest one for the collective."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or world == 1:
        return local
    shards = all_shards(H, world)
    hmax = max(b - a for a, b in shards)
    pad = torch.zeros((hmax,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    return torch.cat([bufs[r][: b - a] for r, (a, b) in enumerate(shards)], dim=0)


def gather_sampled_heads(local, heads, H: int, world: int, rank: int):
    """The full tensors of a few global heads (e.g. outputs [N, d] of heads 0 and H-1) from
    whichever rank owns them: `local` is this rank's [h1-h0, ...] shard. Returns {h: tensor}
    on every rank (an all-gather of a [len(heads), ...] buffer the owners fill)."""
    import torch
    import torch.distributed as dist
    h0, h1 = head_range(H, world, rank)
    buf = torch.zeros((len(heads),) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    for n, h in enumerate(heads):
        if h0 <= h < h1:
            buf[n] = local[h - h0]
    if not (dist.is_available() and dist.is_initialized()) or world == 1:
        return {h: buf[n] for n, h in enumerate(heads)}
    bufs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf)
    owner = {h: next(r for r, (a, b) in enumerate(all_shards(H, world)) if a <= h < b) for h in heads}
    return {h: bufs[owner[h]][n] for n, h in enumerate(heads)}


def gather_outputs(out, device=None):
    """All-gather every rank's output shard (equal shapes) -- verification only."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return [out]
    bufs = [torch.empty_like(out) for _ in range(dist.get_world_size())]
    dist.all_gather(bufs, out.contiguous())
    return bufs
