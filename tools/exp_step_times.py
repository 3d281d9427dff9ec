"""Per-step device times of the bench's flushed headline loop (diagnosis of
the dependence of the mean on --steps)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1112_5239_b200 as P  # noqa: E402
import workloads as W  # noqa: E402
from bench import L2Flush  # noqa: E402

S, n = 2**20, 128
g = P.ChaoticPRNG(W.SEEDS[0], S, P.V1)
out = torch.empty((S, n), dtype=torch.int32, device="cuda")
stream = torch.cuda.current_stream()
flush = L2Flush(torch, torch.device("cuda"))
res = {}
for mode in ("idle_gap", "hot"):
    for _ in range(10):
        g.generate(n, out=out)
    torch.cuda.synchronize()
    if mode == "idle_gap":
        time.sleep(0.2)  # the GPU idles (like NVML init / Python work before the timed loop)
    else:
        for k in range(5):
            flush(k)
            g.generate(n, out=out)
        torch.cuda.synchronize()
    K = 30
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    fev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for k in range(K):
        fev[k][0].record(stream)
        flush(k)
        fev[k][1].record(stream)
        ev[k][0].record(stream)
        g.generate(n, out=out)
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    res[mode] = {"gen_us": [round(a.elapsed_time(b) * 1e3, 1) for a, b in ev],
                 "flush_us": [round(a.elapsed_time(b) * 1e3, 1) for a, b in fev]}
print(json.dumps(res))
