"""V0 with a few streams and long sequences: the split jump-ahead path
(<= 16 streams) against the one-thread-per-stream kernel (CIPRNG_V0_JUMP=0)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1112_5239_b200 as P

torch.cuda.set_device(0)
res = {}
for S, n in ((1, 10**6), (4, 10**6), (16, 10**6), (16, 4 * 10**6)):
    row = {}
    for jump in ("1", "0"):
        os.environ["CIPRNG_V0_JUMP"] = jump
        g = P.ChaoticPRNG(1, S, P.V0)
        out = torch.empty((S, n), dtype=torch.int32, device="cuda")
        for _ in range(3):
            g.generate(n, out=out)
        reps = 20 if jump == "1" else 2
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            g.generate(n, out=out)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        row["jump" if jump == "1" else "one_thread"] = {"ms": ms, "numbers_per_s": S * n / ms * 1e3,
                                                        "path": int(g.info().store_path)}
        g.close()
    res[f"{S}x{n}"] = row
print(json.dumps(res))
