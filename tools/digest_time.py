import torch, time, json, sys
sys.path.insert(0, '.')
import paper_1112_5239_b200 as P
torch.cuda.set_device(0)
S, n = 2**23, 256
out = torch.empty((S, n), dtype=torch.int32, device='cuda')
g = P.ChaoticPRNG(1, S, P.V1)
g.generate(n, out=out)
acc = torch.zeros(1, dtype=torch.int64, device='cuda')
for _ in range(3): P.digest(out, 0, acc)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 20
e0.record()
for _ in range(K): P.digest(out, 0, acc)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / K
print(json.dumps({"digest_ms_8GiB": ms, "TBps": out.numel() * 4 / ms / 1e9}))
