"""World-size-2 tests of the multi-GPU host logic on CPU (gloo backend).

Each rank takes its shard of a batch, computes it (here with the CPU oracle,
standing in for a GPU rank's kernel: the test is about the sharding, the
max-over-ranks timing reduction and the gather), and gathers to rank 0; the
gathered e^A and (m, s) must equal the unsharded computation bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1710_10989_b200.sharding import shard_range


def test_shard_ranges_cover_and_partition():
    for total in (0, 1, 7, 262144, 262145):
        for world in (1, 2, 3, 4, 8):
            shards = [shard_range(r, world, total) for r in range(world)]
            assert sum(s.count for s in shards) == total
            pos = 0
            for s in shards:
                assert s.b0 == pos
                pos += s.count
            assert max(s.count for s in shards) - min(s.count for s in shards) <= 1
    w = [shard_range(r, 4, 1000, weak=True) for r in range(4)]
    assert [s.b0 for s in w] == [0, 1000, 2000, 3000] and all(s.count == 1000 for s in w)
    with pytest.raises(ValueError):
        shard_range(2, 2, 10)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, total, q):
    import torch
    import torch.distributed as dist

    from oracle.oracle import Oracle
    from paper_1710_10989_b200 import workloads
    from paper_1710_10989_b200.sharding import gather_to_root, max_over_ranks, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = shard_range(rank, world, total)
        a = workloads.generate("cfg2", sh.b0, sh.count)
        r = Oracle().expm_batch(a)
        counts = [shard_range(k, world, total).count for k in range(world)]
        out = gather_to_root(torch.from_numpy(r.out), counts)
        deg = gather_to_root(torch.from_numpy(r.degree), counts)
        s = gather_to_root(torch.from_numpy(r.s), counts)
        t = max_over_ranks(float(rank + 1))
        if rank == 0:
            q.put((out.numpy(), deg.numpy(), s.numpy(), t))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("total", [1000, 1001])
def test_gloo_world2_shard_gather_equals_single(total):
    from oracle.oracle import Oracle
    from paper_1710_10989_b200 import workloads

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    out, deg, s, t = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = Oracle().expm_batch(workloads.generate("cfg2", 0, total))
    assert np.array_equal(out.view(np.uint64), ref.out.view(np.uint64))
    assert np.array_equal(deg, ref.degree) and np.array_equal(s, ref.s)
    assert t == 2.0  # max over ranks of (rank + 1)
