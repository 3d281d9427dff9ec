"""Small driver for ncu captures: a few calls of one workload through the
C-ABI.  Usage: python tools/prof_kernels.py {v1|v1direct|v2|v0|v3|v4|consume|consume_v0|consume_v2|consume_v3|battery|cbg|alg1|c1|digest} [calls]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1112_5239_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "v1"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 4
seed = W.SEEDS[0]
if which == "v1smem":
    os.environ["CIPRNG_V1_SMEM_STG"] = "1"
    which = "v1direct"
if which in ("v1", "v1direct"):
    S, n = 2**20, 128
    g = P.ChaoticPRNG(seed, S, P.V1, store_path=P.STORE_DIRECT if which == "v1direct" else P.STORE_TMA)
    out = torch.empty((S, n), dtype=torch.int32, device="cuda")
    for _ in range(calls):
        g.generate(n, out=out)
elif which == "v2":
    S, n = 2**20, 64
    g = P.ChaoticPRNG(seed, S, P.V2)
    out = torch.empty((S, n), dtype=torch.int32, device="cuda")
    for _ in range(calls):
        g.generate(n, out=out)
elif which == "v0":
    S, n = 2**20, 128
    g = P.ChaoticPRNG(seed, S, P.V0)
    out = torch.empty((S, n), dtype=torch.int32, device="cuda")
    for _ in range(calls):
        g.generate(n, out=out)
elif which in ("v3", "v4"):
    S, n = 2**20, 128
    g = P.ChaoticPRNG(seed, S, P.V3 if which == "v3" else P.V4)
    out = torch.empty((S, n), dtype=torch.int32, device="cuda")
    for _ in range(calls):
        g.generate(n, out=out)
elif which == "battery":
    S, n = 2**20, 1024
    g = P.ChaoticPRNG(seed, S, P.V1)
    st = torch.zeros(P.N_BATTERY, dtype=torch.int64, device="cuda")
    for _ in range(calls):
        g.battery(n, st)
elif which == "cbg":
    from paper_1112_5239_b200 import bg as BG

    Bm, L = 2**18, 1024
    N = torch.full((Bm,), 3037000493 * 3037000453 % (2**62), dtype=torch.int64, device="cuda") | 1
    r = torch.randint(2, 2**30, (Bm,), dtype=torch.int64, device="cuda")
    m = torch.randint(0, 256, (Bm, L), dtype=torch.uint8, device="cuda")
    for _ in range(calls):
        BG.encrypt(True, N, r, m)
elif which == "alg1":
    from paper_1112_5239_b200 import chaos as CH

    z = torch.randint(1, 2**31, (2**20,), dtype=torch.int32, device="cuda")
    x = torch.zeros(2**20, dtype=torch.int32, device="cuda")
    for _ in range(calls):
        CH.alg1_generate(32, 8, z, x, 64)
elif which == "c1":
    n = 10**6
    g = P.ChaoticPRNG(0, 1, P.V0, paper_defaults=True)
    out = torch.empty((1, n), dtype=torch.int32, device="cuda")
    for _ in range(calls):
        g.generate(n, out=out)
elif which == "digest":
    S, n = 2**23, 256
    out = torch.empty((S, n), dtype=torch.int32, device="cuda")
    g = P.ChaoticPRNG(seed, S, P.V1)
    g.generate(n, out=out)
    for _ in range(calls):
        P.digest(out)
elif which in ("consume", "consume_v0", "consume_v2", "consume_v3"):
    S, n = 2**20, 1024
    var = {"consume": P.V1, "consume_v0": P.V0, "consume_v2": P.V2, "consume_v3": P.V3}[which]
    g = P.ChaoticPRNG(seed, S, var)
    st = torch.zeros(P.N_STATS, dtype=torch.int64, device="cuda")
    for _ in range(calls):
        g.consume(n, st)
torch.cuda.synchronize()
print("done", which)
