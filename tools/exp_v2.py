"""V2/V4 store timing with and without an L2 flush between calls, evict-first on/off."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1112_5239_b200 as P  # noqa: E402

res = {}
dev = torch.device("cuda", 0)
scratch = torch.empty(64 * 2**20, dtype=torch.int32, device=dev)
stream = torch.cuda.current_stream()
for var, S, n in ((P.V2, 2**20, 64), (P.V4, 2**20, 128), (P.V0, 2**20, 128)):
    g = P.ChaoticPRNG(1, S, var)
    out = torch.empty((S, n), dtype=torch.int32, device=dev)
    for _ in range(3):
        g.generate(n, out=out)
    for flush in (0, 1):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
        torch.cuda.synchronize()
        for k in range(20):
            if flush:
                scratch.fill_(k)
            ev[k][0].record(stream)
            g.generate(n, out=out)
            ev[k][1].record(stream)
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in ev) / 20
        res[f"v{var}_flush{flush}"] = S * n / (ms / 1e3)
    g.close()
print(json.dumps(res))
