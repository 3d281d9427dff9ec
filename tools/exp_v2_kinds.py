"""V2 (C3: 2^20 streams x 64, store) per kernel instantiation (CIPRNG_V2_KIND,
gen_v2.cu): bit-exact check against the oracle on a small case, then
numbers/s with the bench's L2 flush before every call.  One subprocess per
kind (the kind is read at prng_create)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, sys, numpy as np, torch
sys.path.insert(0, ROOT)
import paper_1112_5239_b200 as P, oracle as O
from bench import L2Flush
seed = 0x0123456789ABCDEF
g = P.ChaoticPRNG(seed, 4096, P.V2)
st = O.init_states(P.V2, seed, 0, 4096)
ok = True
for n in (64, 7):
    ok &= bool(np.array_equal(P.as_u32(g.generate(n)), O.generate(P.V2, st, n)))
g.close()
S, n, K = 2**20, 64, 40
g = P.ChaoticPRNG(seed, S, P.V2)
out = torch.empty((S, n), dtype=torch.int32, device="cuda")
fl = L2Flush(torch, torch.device("cuda"))
for _ in range(5): g.generate(n, out=out)
stream = torch.cuda.current_stream()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
for k in range(K):
    fl(k); ev[k][0].record(stream); g.generate(n, out=out); ev[k][1].record(stream)
torch.cuda.synchronize()
ms = sum(a.elapsed_time(b) for a, b in ev) / K
print(json.dumps({"bit_exact": ok, "numbers_per_s": S * n / (ms / 1e3), "ms": ms}))
'''.replace("ROOT", repr(ROOT))
res = {}
kinds = [int(k) for k in sys.argv[1:]] or list(range(11))
for rep in range(2):
    for kind in kinds:
        env = dict(os.environ, CIPRNG_V2_KIND=str(kind))
        r = subprocess.run([sys.executable, "-c", CHILD], capture_output=True, text=True, env=env, cwd=ROOT, timeout=600)
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        res[f"kind{kind}_rep{rep}"] = json.loads(line[-1]) if line else {"error": r.stderr[-500:]}
print(json.dumps(res, indent=1))
