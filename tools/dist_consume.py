"""Fused-consumer run over the process group (BASELINE configs[4] shape):
each rank consumes its shard of the stream space on its own GPU, then one
NCCL all-reduce of the 258 u64 statistics.

  torchrun --nproc-per-node G --master-addr 127.0.0.1 tools/dist_consume.py \
      [--streams 8388608] [--n 1024] [--calls 16] [--variant 1]

Rank 0 prints JSON: stats digest, pi estimate, chi-square p of the top-byte
histogram, consumer throughput (max over ranks, CUDA events), stats list.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1112_5239_b200 as P  # noqa: E402
import workloads as W  # noqa: E402
from paper_1112_5239_b200.dist import allreduce_sum_, shard_range  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--streams", type=int, default=W.CONFIGS["C5"]["n_streams"])
    ap.add_argument("--rounds", type=int, default=W.CONFIGS["C5"]["n"])
    ap.add_argument("--calls", type=int, default=W.CONFIGS["C5"]["calls"])
    ap.add_argument("--variant", type=int, default=1)
    ap.add_argument("--seed", type=int, default=W.SEEDS[0])
    args = ap.parse_args()
    lr = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(lr)
    dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
    ws, rk = dist.get_world_size(), dist.get_rank()
    first, n_local = shard_range(args.streams, ws, rk)
    g = P.ChaoticPRNG(args.seed, args.streams, args.variant, shard=(first, n_local))
    stats = torch.zeros(P.N_STATS, dtype=torch.int64, device="cuda")
    g.consume(2, torch.zeros_like(stats))  # warm-up on a scratch buffer (state advances: re-create)
    g.close()
    g = P.ChaoticPRNG(args.seed, args.streams, args.variant, shard=(first, n_local))
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.calls):
        g.consume(args.rounds, stats)
    allreduce_sum_(stats)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / 1e3], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    s = P.as_u64(stats)
    if rk == 0:
        from scipy import stats as sst

        inside, pairs = int(s[0]), int(s[1])
        p = math.pi / 4
        hist = s[2:].astype(np.float64)
        exp = hist.sum() / 256
        chi2 = float(((hist - exp) ** 2 / exp).sum())
        print(json.dumps({
            "world_size": ws, "variant": args.variant, "streams": args.streams, "n": args.rounds, "calls": args.calls,
            "numbers": args.streams * args.rounds * args.calls,
            "seconds_max_over_ranks": float(t.item()),
            "numbers_per_s": args.streams * args.rounds * args.calls / float(t.item()),
            "pi_hat": 4 * inside / pairs, "pi_z": (inside / pairs - p) / math.sqrt(p * (1 - p) / pairs),
            "hist_chi2_p": float(sst.chi2.sf(chi2, 255)),
            "stats": [int(v) for v in s],
        }))
    g.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
