"""How the L2 flush between timed calls is done changes what the timed V1 C2
call pays for: a 256 MiB write leaves up to ~126 MB of DIRTY flush lines in
L2 that get written back inside the next timed call.  Compare (a) write
flush, (b) write flush then a 256 MiB read (dirty lines written back before
the timer starts; L2 ends full of clean unrelated lines), (c) read-only
flush, (d) no flush.  Numbers/s per mode, 100 calls each."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1112_5239_b200 as P  # noqa: E402

S, n, K = 2**20, 128, 100
g = P.ChaoticPRNG(0x0123456789ABCDEF, S, P.V1)
out = torch.empty((S, n), dtype=torch.int32, device="cuda")
wbuf = torch.empty(64 * 2**20, dtype=torch.int32, device="cuda")
rbuf = torch.ones(64 * 2**20, dtype=torch.int32, device="cuda")
acc = torch.empty((), dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream()


def flush(mode, k):
    if mode in ("write", "write+read"):
        wbuf.fill_(k)
    if mode in ("write+read", "read"):
        acc.copy_(torch.amax(rbuf))


res = {}
for rep in range(2):
    for mode in ("write", "write+read", "read", "none"):
        for _ in range(5):
            g.generate(n, out=out)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        for k in range(K):
            flush(mode, k)
            ev[k][0].record(st)
            g.generate(n, out=out)
            ev[k][1].record(st)
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in ev) / K
        res[f"{mode}_rep{rep}"] = {"numbers_per_s": S * n / (ms / 1e3), "ms": ms}
print(json.dumps(res, indent=1))
