"""Shared helpers of the GPU parity tests: run the same seeded workload
through the C-ABI (CUDA path) and through the oracle, return comparable
numpy arrays.  Imports both sides; neither side imports the other."""
from __future__ import annotations

import numpy as np
import torch

import oracle as O
import paper_1112_5239_b200 as P


def gpu_run(variant, seed, S, ns, *, first=0, comb_size=None, comb=None, paper_defaults=False,
            store_path=P.STORE_AUTO, out_offset_words=0):
    """Create a handle, run generate() for each n in ns; return (outs, planes, info)."""
    g = P.ChaoticPRNG(seed, first + S, variant, shard=(first, S), comb_size=comb_size, comb=comb,
                      paper_defaults=paper_defaults, store_path=store_path)
    outs = []
    for n in ns:
        if out_offset_words:
            buf = torch.empty(S * n + out_offset_words, dtype=torch.int32, device="cuda")
            view = buf[out_offset_words:]
            g.generate(n, out=view)
            outs.append(P.as_u32(view).reshape(S, n))
        else:
            outs.append(P.as_u32(g.generate(n)))
    torch.cuda.synchronize()
    planes = g.get_state()
    info = g.info()
    g.close()
    return outs, planes, info


def oracle_run(variant, seed, S, ns, *, first=0, comb_size=32, comb=None, paper_defaults=False):
    st = O.init_states(variant, seed, first, S, paper_defaults=paper_defaults)
    outs = [O.generate(variant, st, n, comb_size=comb_size, comb=comb) for n in ns]
    return outs, O.state_planes(variant, st)


def first_mismatch(a: np.ndarray, b: np.ndarray) -> str:
    if a.shape != b.shape:
        return f"shape {a.shape} vs {b.shape}"
    bad = np.argwhere(a != b)
    if bad.size == 0:
        return "equal"
    idx = tuple(bad[0])
    return f"{len(bad)} mismatches, first at {idx}: gpu={a[idx]} oracle={b[idx]}"
