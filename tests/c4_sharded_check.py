"""BASELINE configs[3]: stream-sharded generation of ~10^12 numbers, output
identical at every GPU count.

  python tests/c4_sharded_check.py [--calls 466] [--gpus-simulated 1,2,4,8] [--verify-groups 64]

V1, 2^23 streams x 256 numbers per call, 466 calls = 1,000,727,379,968
numbers.  For each shard count G the stream space is split with
dist.shard_range; the shards run one after another on this GPU (or, under
torchrun, rank r runs shard r of G = world size).  Every call's output is
digested on device (prng_digest, position-aware, additive across shards) and
the per-call digest list must be identical for every G.  Then sampled
32-stream groups are replayed by the oracle through all calls and compared
word for word with the GPU output of the same groups (regenerated from their
own shard handles).  Writes JSON to stdout.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1112_5239_b200 as P  # noqa: E402
import workloads as W  # noqa: E402
from paper_1112_5239_b200.dist import shard_range  # noqa: E402


def run_shards(G: int, S: int, n: int, calls: int, seed: int):
    """Digest list of `calls` calls over S streams split into G shards."""
    digests = np.zeros(calls, dtype=np.uint64)
    gpu_s = gen_s = 0.0
    for r in range(G):
        first, n_local = shard_range(S, G, r)
        g = P.ChaoticPRNG(seed, S, P.V1, shard=(first, n_local))
        out = torch.empty((n_local, n), dtype=torch.int32, device="cuda")
        acc = torch.zeros(calls, dtype=torch.int64, device="cuda")
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for c in range(calls):
            g.generate(n, out=out)
            P.digest(out, first_stream=first, acc=acc[c:c + 1])
        ev1.record()
        torch.cuda.synchronize()
        gpu_s += ev0.elapsed_time(ev1) / 1e3
        digests += P.as_u64(acc)  # uint64 wrap-around == mod 2^64
        # generation alone (the same shard handle continues: calls+1.., work
        # identical in shape), back-to-back launches
        ev0.record()
        for c in range(calls):
            g.generate(n, out=out)
        ev1.record()
        torch.cuda.synchronize()
        gen_s += ev0.elapsed_time(ev1) / 1e3
        g.close()
        del out
    return digests, gpu_s, gen_s


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--calls", type=int, default=W.CONFIGS["C4"]["calls"])
    ap.add_argument("--streams", type=int, default=W.CONFIGS["C4"]["n_streams"])
    ap.add_argument("--n", type=int, default=W.CONFIGS["C4"]["n"])
    ap.add_argument("--gpus-simulated", default="1,2,4,8")
    ap.add_argument("--verify-groups", type=int, default=64)
    args = ap.parse_args()
    seed = W.SEEDS[0]
    S, n, calls = args.streams, args.n, args.calls
    res = {"workload": f"C4: V1, {S} streams x {n} x {calls} calls", "numbers": S * n * calls, "per_G": {}}
    ref = None
    for G in [int(x) for x in args.gpus_simulated.split(",")]:
        d, gpu_s, gen_s = run_shards(G, S, n, calls, seed)
        same = ref is None or bool(np.array_equal(d, ref))
        ref = d if ref is None else ref
        res["per_G"][G] = {"gpu_seconds_incl_digest": gpu_s, "digests_equal_G1": same,
                           "generate_seconds_sum_over_shards": gen_s,
                           "generate_numbers_per_s_per_gpu": S * n * calls / gen_s,
                           "first_digests": [int(v) for v in d[:3]]}
    # oracle replay of sampled groups through all calls
    import oracle as O

    gen = W.rng(4)
    groups = np.sort(gen.choice(S // 32, args.verify_groups, replace=False))
    t0 = time.perf_counter()
    ok = True
    for gr in groups:
        first = int(gr) * 32
        g = P.ChaoticPRNG(seed, S, P.V1, shard=(first, 32), comb_size=32)
        st = O.init_states(O.V1, seed, first, 32)
        for c in range(calls):
            a = P.as_u32(g.generate(n))
            b = O.generate(O.V1, st, n)
            if not np.array_equal(a, b):
                ok = False
                break
        g.close()
        if not ok:
            break
    res["oracle_replay"] = {"groups": int(args.verify_groups), "calls": calls, "bit_exact": ok,
                            "seconds": time.perf_counter() - t0}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
