"""Multi-GPU plumbing (one process per GPU, torch.distributed).

SURVEY s8(e): the path shards naturally -- units are 32-stream combination
groups, a group never exchanges data with another, and the state of global
stream s is a pure function of (seed, s) (reading Q11), so rank r simply owns
a contiguous range of whole groups.  The store path has NO collective; the
only exchange step is the consumer statistics (and verification digests),
summed with one all-reduce (NCCL on GPUs, gloo in the CPU tests).  Integer
sums are order-independent, so results are bit-identical at any GPU count.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_streams: int, world_size: int, rank: int, align: int = 32) -> tuple[int, int]:
    """Contiguous stream range [first, first + n_local) of `rank`: whole
    groups of `align` streams, as even as possible (the first n_groups %
    world_size ranks get one extra group)."""
    if n_streams % align:
        raise ValueError(f"n_streams={n_streams} is not a multiple of the group size {align}")
    if not 0 <= rank < world_size:
        raise ValueError("rank out of range")
    groups = n_streams // align
    base, extra = divmod(groups, world_size)
    first_g = rank * base + min(rank, extra)
    n_g = base + (1 if rank < extra else 0)
    return first_g * align, n_g * align


# number of all-reduces that actually ran a collective (world size > 1) in
# this process -- lets tests assert the exchange step really executed
COLLECTIVES_RUN = 0


def allreduce_sum_(t: torch.Tensor, group=None) -> torch.Tensor:
    """In-place SUM all-reduce of an int64 tensor (u64 bit patterns wrap the
    same way under two's complement addition).  No-op without a process group
    or at world size 1 (there is nothing to exchange)."""
    global COLLECTIVES_RUN
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        COLLECTIVES_RUN += 1
    return t


def sharded_consume(seed: int, n_streams: int, variant: int, n: int, calls: int, *, group=None,
                    stats: torch.Tensor | None = None) -> torch.Tensor:
    """Consumer mode over the global stream space, sharded over the process
    group: each rank runs its own streams on its own GPU (prng_consume), then
    one all-reduce of the 258 u64 statistics (the a7 row of SURVEY s8(a))."""
    import paper_1112_5239_b200 as P

    ws = dist.get_world_size(group) if dist.is_initialized() else 1
    rk = dist.get_rank(group) if dist.is_initialized() else 0
    first, n_local = shard_range(n_streams, ws, rk)
    g = P.ChaoticPRNG(seed, n_streams, variant, shard=(first, n_local))
    if stats is None:
        stats = torch.zeros(P.N_STATS, dtype=torch.int64, device=g.device)
    for _ in range(calls):
        g.consume(n, stats)
    g.close()
    return allreduce_sum_(stats, group)


def sharded_digests(seed: int, n_streams: int, variant: int, n: int, calls: int, *, group=None) -> list[int]:
    """Store mode over the global stream space: per call, each rank generates
    its shard and digests it (position-aware, reading Q28); the digests are
    summed across ranks.  The list is identical at every GPU count."""
    import paper_1112_5239_b200 as P

    ws = dist.get_world_size(group) if dist.is_initialized() else 1
    rk = dist.get_rank(group) if dist.is_initialized() else 0
    first, n_local = shard_range(n_streams, ws, rk)
    g = P.ChaoticPRNG(seed, n_streams, variant, shard=(first, n_local))
    out = torch.empty((n_local, n), dtype=torch.int32, device=g.device)
    res = []
    for _ in range(calls):
        g.generate(n, out=out)
        d = P.digest(out, first_stream=first)
        res.append(int(allreduce_sum_(d, group).item()) % 2**64)
    g.close()
    return res
