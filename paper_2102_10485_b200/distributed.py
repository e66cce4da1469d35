"""Label sharding across the GPUs of one box (the B200 form of
train_distributed, /root/reference/proj/src/partition.cpp:116-180).

Labels never exchange gradients, so the path shards into
independent label blocks: rank r of P owns labels [shard_begin(n, P, r),
shard_begin(n, P, r+1)) — balanced contiguous blocks whose sizes differ by at
most one.  There is no collective inside the training loop; the only
communication is one gather at the end: 64 generated samples per label plus
per-label loss statistics, over NCCL (torch.distributed) when the ranks are
GPUs, over gloo in the CPU tests.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_labels: int, world: int, rank: int) -> range:
    """Contiguous block of labels owned by `rank` (mirrors pg_shard_begin)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid rank / world size")
    begin = (rank * n_labels) // world
    end = ((rank + 1) * n_labels) // world
    return range(begin, end)


def gather_to_root(t: torch.Tensor, n_labels: int, world: int, rank: int) -> torch.Tensor | None:
    """Gather per-rank label blocks [labels_of_rank, ...] into [n_labels, ...]
    on rank 0 (ranks may own different label counts: pads to the largest
    block, gathers, then strips).  Returns the full tensor on rank 0, None
    elsewhere."""
    if world == 1:
        return t
    own = len(shard_range(n_labels, world, rank))
    biggest = max(len(shard_range(n_labels, world, r)) for r in range(world))
    pad = torch.zeros((biggest - own,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    sendbuf = torch.cat([t, pad]) if biggest > own else t.contiguous()
    if rank == 0:
        recv = [torch.empty_like(sendbuf) for _ in range(world)]
        dist.gather(sendbuf, recv, dst=0)
        parts = [recv[r][:len(shard_range(n_labels, world, r))] for r in range(world)]
        return torch.cat(parts)
    dist.gather(sendbuf, None, dst=0)
    return None


def max_over_ranks(value: float, device: str | torch.device = "cpu") -> float:
    """Max of a scalar over ranks (the timing rule: a step takes as long as
    its slowest rank)."""
    if not dist.is_available() or not dist.is_initialized():
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
