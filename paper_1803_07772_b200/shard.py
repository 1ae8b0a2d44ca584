"""Multi-GPU sharding of independent channel realisations.

Instances never interact, so a batch is split into contiguous draw ranges,
one per rank (one process per GPU), with no collective on the data path.
Seeds stay global (draw index), so the split never changes any result.  The
only collectives are optional and outside the solve: the max-over-ranks
device time (timing) and one gather of per-instance scalars to rank 0.
Works with the "nccl" backend on GPUs and "gloo" on CPU tensors (tests).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

SCALARS = ("ee", "sum_rate", "total_power", "final_e", "outer_iters", "rounds", "sweeps",
           "status", "feasible")


def shard_range(rank: int, world: int, total: int) -> range:
    """Contiguous block of draws for `rank` (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    q, r = divmod(total, world)
    lo = rank * q + min(rank, r)
    return range(lo, lo + q + (1 if rank < r else 0))


def weak_range(rank: int, per_rank: int, offset: int = 0) -> range:
    """Weak scaling: every rank solves its own `per_rank` draws."""
    return range(offset + rank * per_rank, offset + (rank + 1) * per_rank)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (the device time of the timed region)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_scalars(outs: dict, device=None) -> dict | None:
    """Gather the per-instance scalar outputs of every rank to rank 0, in rank
    order (= draw order for `shard_range` / `weak_range`).  Returns the
    concatenated dict on rank 0 and None elsewhere."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return {k: outs[k] for k in SCALARS if k in outs}
    world, rank = dist.get_world_size(), dist.get_rank()
    res = {}
    for k in SCALARS:
        if k not in outs:
            continue
        t = outs[k].to(device=device, dtype=torch.float64).contiguous()
        n = torch.tensor([t.numel()], dtype=torch.int64, device=device)
        sizes = [torch.zeros_like(n) for _ in range(world)]
        dist.all_gather(sizes, n)
        mx = int(max(s.item() for s in sizes))
        pad = torch.zeros(mx, dtype=torch.float64, device=device)
        pad[:t.numel()] = t
        bufs = [torch.zeros(mx, dtype=torch.float64, device=device) for _ in range(world)]
        dist.all_gather(bufs, pad)
        if rank == 0:
            res[k] = torch.cat([b[:int(s.item())] for b, s in zip(bufs, sizes)])
    return res if rank == 0 else None
