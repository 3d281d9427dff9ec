"""Sharded consumer + verification digests over the process group (the a7
row; BASELINE configs[4] shape by default): each rank consumes its shard of
the stream space on its own GPU through dist.sharded_consume (prng_consume,
then one SUM all-reduce of the 258 u64 statistics), then, from fresh
handles, runs dist.sharded_digests (prng_generate + prng_digest per call,
digests summed across ranks).

  torchrun --nproc-per-node G --master-addr 127.0.0.1 tools/dist_consume.py \
      [--streams 8388608] [--rounds 1024] [--calls 16] [--variant 1] \
      [--backend nccl|gloo] [--digest-calls 0]

gloo lets several ranks share one GPU (CUDA tensors, host-staged reduce);
NCCL needs one GPU per rank.  Rank 0 prints JSON: the reduced statistics,
the digest list, pi estimate, chi-square p of the top-byte histogram,
consumer throughput (max over ranks, CUDA events) and how many all-reduces
actually ran a collective on this rank.
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
import paper_1112_5239_b200.dist as D  # noqa: E402
import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--streams", type=int, default=W.CONFIGS["C5"]["n_streams"])
    ap.add_argument("--rounds", type=int, default=W.CONFIGS["C5"]["n"])
    ap.add_argument("--calls", type=int, default=W.CONFIGS["C5"]["calls"])
    ap.add_argument("--variant", type=int, default=1)
    ap.add_argument("--seed", type=int, default=W.SEEDS[0])
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--digest-calls", type=int, default=0)
    args = ap.parse_args()
    lr = int(os.environ.get("LOCAL_RANK", "0"))
    dev = lr % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    if args.backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group("gloo")
    ws, rk = dist.get_world_size(), dist.get_rank()
    nccl_version = ".".join(map(str, torch.cuda.nccl.version())) if args.backend == "nccl" else None
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    stats = D.sharded_consume(args.seed, args.streams, args.variant, args.rounds, args.calls)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / 1e3], dtype=torch.float64, device="cuda")
    if args.backend == "gloo":
        t = t.cpu()
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    digs = D.sharded_digests(args.seed, args.streams, args.variant, args.rounds, args.digest_calls) \
        if args.digest_calls else []
    s = P.as_u64(stats)
    if rk == 0:
        from scipy import stats as sst

        inside, pairs = int(s[0]), int(s[1])
        p = math.pi / 4
        hist = s[2:].astype(np.float64)
        exp = hist.sum() / 256
        chi2 = float(((hist - exp) ** 2 / exp).sum())
        print(json.dumps({
            "world_size": ws, "backend": args.backend, "nccl_version": nccl_version, "variant": args.variant,
            "seed": args.seed, "streams": args.streams, "n": args.rounds, "calls": args.calls,
            "numbers": args.streams * args.rounds * args.calls,
            "seconds_max_over_ranks": float(t.item()),
            "numbers_per_s": args.streams * args.rounds * args.calls / float(t.item()),
            "pi_hat": 4 * inside / pairs, "pi_z": (inside / pairs - p) / math.sqrt(p * (1 - p) / pairs),
            "hist_chi2_p": float(sst.chi2.sf(chi2, 255)),
            "collectives_run": D.COLLECTIVES_RUN,
            "stats": [int(v) for v in s], "digests": digs,
        }))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
