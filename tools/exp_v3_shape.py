"""V3 store (2^20 streams x 128, L2 flushed) for the library as built (box
shape knobs CIPRNG_V3_COLS / CIPRNG_V3_WPB via CIPRNG_NVCC_EXTRA), after a
bit-exact check against the oracle on a small case."""
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
g = P.ChaoticPRNG(seed, 4096 + 64, P.V3, store_path=P.STORE_TMA)
st = O.init_states(P.V3, seed, 0, 4096 + 64)
ok = True
for n in (128, 36, 200):
    ok &= bool(np.array_equal(P.as_u32(g.generate(n)), O.generate(P.V3, st, n)))
g.close()
S, n, K = 2**20, 128, 40
g = P.ChaoticPRNG(seed, S, P.V3)
out = torch.empty((S, n), dtype=torch.int32, device="cuda")
fl = L2Flush(torch, torch.device("cuda"))
for _ in range(5):
    g.generate(n, out=out)
stream = torch.cuda.current_stream()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
for k in range(K):
    fl(k)
    ev[k][0].record(stream)
    g.generate(n, out=out)
    ev[k][1].record(stream)
torch.cuda.synchronize()
ms = sum(a.elapsed_time(b) for a, b in ev) / K
print(json.dumps({"build": os.environ.get("CIPRNG_NVCC_EXTRA", ""), "bit_exact": ok, "path": g.info().store_path,
                  "numbers_per_s": S * n / (ms / 1e3)}))
