"""V1 store throughput when no TMA descriptor applies (n % 4 != 0, or an
output 4 bytes off 16-byte alignment): AUTO (staged shared-memory +
coalesced STG) vs DIRECT (per-lane stores), L2 flushed before each call."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1112_5239_b200 as P  # noqa: E402

S = 2**20
res = {}
scratch = torch.empty(64 * 2**20, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream()
for n, off in ((127, 0), (128, 1), (128, 0)):
    for name, sp in (("auto", P.STORE_AUTO), ("direct", P.STORE_DIRECT)):
        g = P.ChaoticPRNG(1, S, P.V1, store_path=sp)
        buf = torch.empty(S * n + 4, dtype=torch.int32, device="cuda")
        out = buf[off:off + S * n]
        for _ in range(3):
            g.generate(n, out=out)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
        for k in range(20):
            scratch.fill_(k)
            ev[k][0].record(st)
            g.generate(n, out=out)
            ev[k][1].record(st)
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in ev) / 20
        res[f"n{n}_off{off}_{name}"] = S * n / (ms / 1e3)
        g.close()
print(json.dumps(res))
