"""Multi-GPU plumbing for batched expm: one process per GPU (torch.distributed),
matrices sharded by contiguous index ranges, no collective on the data path,
one gather of e^A (+ selection records) to rank 0 to collect results, and
device time reduced as the max over ranks.

SURVEY.md section 8(e): matrices are independent, so rank r owns
[b0, b0 + count); a matrix's (m, s) and e^A do not depend on the shard, so the
gathered result equals the single-GPU result bit for bit. The reference's only
parallelism is the OpenMP row split inside one product
(/root/reference/proj/src/kernels.cpp:16-27); splitting the batch by matrix is
this path's own design. The same split is done natively, in one process, by
``mexp_expm_batched_host_multi`` (csrc/capi.cu).
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

    weak=False (the default): `total` matrices split as evenly
    as possible, [k*B/G + min(k, B%G), ...) -- the first total % world ranks
    get one more. weak=True: every rank owns a full batch of `total` matrices
    (global indices [rank * total, (rank + 1) * total)), per-GPU work fixed as
    the GPU count grows.
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


def gather_to_root(local, counts, root: int = 0, out=None):
    """Gather each rank's (count_r, ...) tensor to `root`, concatenated in rank
    order; other ranks get None.

    Grouped point-to-point (``torch.distributed.batch_isend_irecv``: one
    ncclGroupStart/End around every rank's ncclSend to the root and the root's
    ncclRecv from each rank -- NCCL has no ragged gather): the root receives
    straight into its slice of the result, so shards of different lengths
    need no padding and no concatenation copy. ``out`` (root only) may supply
    the (sum(counts), ...) result buffer. Works with NCCL (CUDA tensors) and
    gloo (CPU tensors).
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    rank = dist.get_rank()
    if local.shape[0] != counts[rank]:
        raise ValueError("local shard length differs from counts[rank]")
    local = local.contiguous()
    if rank != root:
        if counts[rank]:
            for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, local, root)]):
                w.wait()
        return None
    total = sum(counts)
    if out is None:
        out = torch.empty((total,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    offs = [sum(counts[:r]) for r in range(world)]
    ops = [dist.P2POp(dist.irecv, out[offs[r]:offs[r] + counts[r]], r)
           for r in range(world) if r != root and counts[r]]
    works = dist.batch_isend_irecv(ops) if ops else []
    out[offs[root]:offs[root] + counts[root]].copy_(local)
    for w in works:
        w.wait()
    return out
