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


def gather_outputs(out, device=None):
    """All-gather every rank's output shard (equal shapes) -- verification only."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return [out]
    bufs = [torch.empty_like(out) for _ in range(dist.get_world_size())]
    dist.all_gather(bufs, out.contiguous())
    return bufs
