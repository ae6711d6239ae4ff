"""Multi-GPU plumbing for batched expm: one process per GPU (torch.distributed),
matrices sharded by contiguous index ranges, no collective on the data path,
one gather of e^A (+ selection records) to rank 0 to collect results, and
device time reduced as the max over ranks.

SURVEY.md section 8(e): matrices are independent, so rank r owns
[b0, b0 + count); a matrix's (m, s) and e^A do not depend on the shard, so the
gathered result equals the single-GPU result bit for bit.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    b0: int       # first global matrix index of this rank
    count: int    # matrices on this rank


def shard_range(rank: int, world: int, total: int, weak: bool = False) -> Shard:
    """Contiguous shard of rank `rank`.

    weak=True: every rank owns a full batch of `total` matrices (global
    indices [rank * total, (rank + 1) * total)) -- per-GPU work fixed as the
    GPU count grows. weak=False: `total` matrices split as evenly as possible
    (the first total % world ranks get one more).
    """
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    if weak:
        return Shard(rank, world, rank * total, total)
    base, extra = divmod(total, world)
    count = base + (1 if rank < extra else 0)
    b0 = rank * base + min(rank, extra)
    return Shard(rank, world, b0, count)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (device time) over all ranks."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_to_root(local, counts, root: int = 0):
    """Gather each rank's (count_r, ...) tensor to `root`, concatenated in rank
    order; other ranks get None. Shards may differ in length: every rank pads
    to the largest count (torch.distributed.gather needs equal shapes) and the
    root trims. Works with NCCL (CUDA tensors) and gloo (CPU tensors).
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    rank = dist.get_rank()
    cmax = max(counts)
    if local.shape[0] < cmax:
        pad = torch.zeros((cmax - local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype,
                          device=local.device)
        send = torch.cat([local, pad])
    else:
        send = local.contiguous()
    if rank == root:
        bufs = [torch.empty_like(send) for _ in range(world)]
        dist.gather(send, bufs, dst=root)
        return torch.cat([b[:c] for b, c in zip(bufs, counts)])
    dist.gather(send, None, dst=root)
    return None
