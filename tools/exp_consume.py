"""C5-shaped V1 consumer timing (2^20 streams x 1024 per call, L2 flushed
before each call) for the library as built -- run once per experiment build
(CIPRNG_NVCC_EXTRA=-DCIPRNG_EXP_...)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1112_5239_b200 as P  # noqa: E402
from bench import L2Flush  # noqa: E402

S, n, K = 2**20, 1024, 20
res = {"build": os.environ.get("CIPRNG_NVCC_EXTRA", "")}
fl = L2Flush(torch, torch.device("cuda"))
st = torch.cuda.current_stream()
for var in (P.V1, P.V3, P.V2, P.V0):
    nn = 64 if var == P.V2 else n
    g = P.ChaoticPRNG(1, S, var)
    stats = torch.zeros(P.N_STATS, dtype=torch.int64, device="cuda")
    for _ in range(3):
        g.consume(nn, stats)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for k in range(K):
        fl(k)
        ev[k][0].record(st)
        g.consume(nn, stats)
        ev[k][1].record(st)
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev) / K
    res[f"v{var}_consume"] = S * nn / (ms / 1e3)
    if var == P.V2:  # also at the bench's C5 shape (n = 1024)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(5)]
        g.consume(n, stats)
        for k in range(5):
            fl(k)
            ev[k][0].record(st)
            g.consume(n, stats)
            ev[k][1].record(st)
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in ev) / 5
        res["v2_consume_1024"] = S * n / (ms / 1e3)
    g.close()
for var in (P.V1, P.V3):  # the NEXT-2 battery (same shape)
    g = P.ChaoticPRNG(1, S, var)
    bst = torch.zeros(P.N_BATTERY, dtype=torch.int64, device="cuda")
    for _ in range(3):
        g.battery(n, bst)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for k in range(K):
        fl(k)
        ev[k][0].record(st)
        g.battery(n, bst)
        ev[k][1].record(st)
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev) / K
    res[f"v{var}_battery"] = S * n / (ms / 1e3)
    g.close()
print(json.dumps(res))
