"""The paper's throughput-vs-threads experiment (PAPER.md P:1015-1060,
Figures "time_xorlike_gpu" and "time_bbs_gpu") re-run on one B200 with this
implementation: 32-bit numbers per second as a function of the number of
streams (= the paper's GPU threads), 2^10 .. 2^23 plus 5M, for

  * the naive xor-like PRNG (Listing 1 per thread = V0),
  * the optimized one (Alg. 4 with xor64 = V3, the paper's "optimized
    versions use the xor64"),
  * Alg. 4 with 32-bit xor128 (V1, the algorithm section's kernel),
  * the BBS PRNG (Alg. 5 = V2),

each in the paper's measurement mode -- numbers not stored,
here the fused consumer (Monte-Carlo pi + histogram, every number used) --
and in store mode (every number written to HBM).  n = 1024 numbers per
stream per call for the consumer (BBS: 256), 128 in store mode (BBS: 64);
back-to-back calls timed with CUDA events (20 calls, after 3 warm-up).

  python tools/fig_threads.py > profiles/<tag>_fig_threads.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1112_5239_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

SIZES = [2**k for k in range(10, 24)] + [5 * 2**20]
ROWS = [  # (name, variant, mode, n)
    ("naive_V0_consume", P.V0, "consume", 1024),
    ("optimized_xor64_V3_consume", P.V3, "consume", 1024),
    ("alg4_xor128_V1_consume", P.V1, "consume", 1024),
    ("bbs_V2_consume", P.V2, "consume", 256),
    ("naive_V0_store", P.V0, "store", 128),
    ("optimized_xor64_V3_store", P.V3, "store", 128),
    ("alg4_xor128_V1_store", P.V1, "store", 128),
    ("bbs_V2_store", P.V2, "store", 64),
]


def measure(variant, mode, S, n, calls=20):
    g = P.ChaoticPRNG(W.SEEDS[0], S, variant)
    if mode == "store":
        out = torch.empty((S, n), dtype=torch.int32, device="cuda")
        fn = lambda: g.generate(n, out=out)  # noqa: E731
    else:
        stats = torch.zeros(P.N_STATS, dtype=torch.int64, device="cuda")
        fn = lambda: g.consume(n, stats)  # noqa: E731
    for _ in range(3):
        fn()
    st = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(st)
    for _ in range(calls):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    g.close()
    return calls * S * n / (a.elapsed_time(b) / 1e3)


def main():
    res = {"what": __doc__.split("\n\n")[0], "unit": "numbers/s", "streams": SIZES, "rows": {}}
    for name, var, mode, n in ROWS:
        res["rows"][name] = {"n": n, "values": [measure(var, mode, S, n) for S in SIZES]}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
