"""C1 jump-kernel phase timing (CIPRNG_NVCC_EXTRA=-DCIPRNG_JUMP_TIMING builds print per-phase globaltimer stamps)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1112_5239_b200 as P
g = P.ChaoticPRNG(0, 1, P.V0, paper_defaults=True)
out = torch.empty((1, 10**6), dtype=torch.int32, device="cuda")
for _ in range(5):
    g.generate(10**6, out=out)
torch.cuda.synchronize()
