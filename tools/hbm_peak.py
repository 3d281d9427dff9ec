"""HBM write / copy bandwidth microbenchmark (context for the V1 store
roofline): torch fill_ (coalesced vector stores, write-only), zero_
(cudaMemsetAsync), copy_ (read+write, the MEASURED_PEAKS method)."""
import json
import sys

import torch

res = {}
for mib in (512, 4096):
    n = mib * 2**20 // 4
    a = torch.empty(n, dtype=torch.int32, device="cuda")
    b = torch.empty(n, dtype=torch.int32, device="cuda")
    for name, fn, bytes_ in (("fill", lambda: a.fill_(7), 4 * n), ("memset", lambda: a.zero_(), 4 * n),
                             ("copy", lambda: b.copy_(a), 8 * n)):
        for _ in range(5):
            fn()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 50
        torch.cuda.synchronize()
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        t = s.elapsed_time(e) / 1e3 / reps
        res[f"{name}_{mib}MiB_GBps"] = bytes_ / t / 1e9
    del a, b
print(json.dumps(res))
