"""V0 / V4 store (2^20 streams x 128, L2 flushed) for the library as built
(CTA shape knobs CIPRNG_V0_* via CIPRNG_NVCC_EXTRA), after a bit-exact check
against the oracle on a small case."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_1112_5239_b200 as P  # noqa: E402
from bench import L2Flush  # noqa: E402

seed = 0x0123456789ABCDEF
res = {"build": os.environ.get("CIPRNG_NVCC_EXTRA", "")}
fl = L2Flush(torch, torch.device("cuda"))
stream = torch.cuda.current_stream()
for var in (P.V0, P.V4):
    g = P.ChaoticPRNG(seed, 1024, var)
    st = O.init_states(var, seed, 0, 1024)
    ok = all(bool(np.array_equal(P.as_u32(g.generate(n)), O.generate(var, st, n))) for n in (40, 7))
    g.close()
    S, n, K = 2**20, 128, 30
    g = P.ChaoticPRNG(seed, S, var)
    out = torch.empty((S, n), dtype=torch.int32, device="cuda")
    for _ in range(3):
        g.generate(n, out=out)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for k in range(K):
        fl(k)
        ev[k][0].record(stream)
        g.generate(n, out=out)
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev) / K
    res[f"v{var}"] = S * n / (ms / 1e3)
    res[f"v{var}_exact"] = ok
    g.close()
print(json.dumps(res))
