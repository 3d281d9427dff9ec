"""Multi-process (gloo, world_size 2, CPU) tests of the sharding host logic:
the partition of the stream space and the statistics / digest all-reduce.
The per-rank compute is the oracle here (no GPU); on GPUs the same
dist.shard_range / allreduce_sum_ run with NCCL around prng_consume."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1112_5239_b200.dist import allreduce_sum_, shard_range


def test_shard_range_partition():
    for S, G in [(64, 2), (96, 2), (2**20, 8), (32 * 7, 3), (32, 4)]:
        ranges = [shard_range(S, G, r) for r in range(G)]
        pos = 0
        for first, n in ranges:
            assert first == pos and first % 32 == 0 and n % 32 == 0
            pos += n
        assert pos == S
        sizes = [n for _, n in ranges]
        assert max(sizes) - min(sizes) <= 32
    with pytest.raises(ValueError):
        shard_range(33, 2, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, variant, S, n, calls, q):
    import oracle as O

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    first, n_local = shard_range(S, ws, rank)
    st = O.init_states(variant, 0xABC, first, n_local)
    stats = np.zeros(258, np.uint64)
    digs = []
    for _ in range(calls):
        out = O.generate(variant, st, n)
        O.stats(out, stats)
        d = torch.tensor([O.digest(out, first)], dtype=torch.uint64).view(torch.int64)
        digs.append(int(allreduce_sum_(d).item()) % 2**64)
    t = torch.from_numpy(stats.view(np.int64).copy())
    allreduce_sum_(t)
    if rank == 0:
        q.put((t.numpy().view(np.uint64).tolist(), digs))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("variant", [0, 1, 2])
def test_gloo_sharded_stats_and_digests_equal_unsharded(variant):
    import oracle as O

    S, n, calls = 96, 10, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, variant, S, n, calls, q)) for r in range(2)]
    for p in procs:
        p.start()
    stats, digs = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    st = O.init_states(variant, 0xABC, 0, S)
    ref = np.zeros(258, np.uint64)
    ref_d = []
    for _ in range(calls):
        out = O.generate(variant, st, n)
        O.stats(out, ref)
        ref_d.append(O.digest(out))
    assert stats == ref.tolist()
    assert digs == ref_d
