"""Algorithm 1 and the chaos / uniformity checks (
PAPER.md P:370-447): thin marshalling over ``prng_alg1_generate`` and
``prng_gamma_check`` (include/ciprng.h)."""
from __future__ import annotations

import ctypes

import torch

from ._lib import check, lib


def _p(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream(stream):
    return ctypes.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)


def alg1_generate(n: int, b: int, z: torch.Tensor, x: torch.Tensor, n_out: int, f: torch.Tensor | None = None,
                  stream=None) -> torch.Tensor:
    """z, x: int32 CUDA [S] (u32 bits), advanced in place -> int32 [S, n_out]."""
    S = z.numel()
    out = torch.empty((S, n_out), dtype=torch.int32, device=z.device)
    check(lib().prng_alg1_generate(_p(f), n, b, _p(z), _p(x), S, n_out, _p(out), _stream(stream)),
          "prng_alg1_generate")
    return out


def gamma_check(n: int, f: torch.Tensor | None = None, device="cuda", stream=None) -> dict:
    scratch = torch.empty(1 << n, dtype=torch.uint8, device=device)
    rep = torch.zeros(3, dtype=torch.int64, device=device)
    check(lib().prng_gamma_check(_p(f), n, _p(scratch), _p(rep), _stream(stream)), "prng_gamma_check")
    r = rep.cpu().tolist()
    V = 1 << n
    return {"reach_from_0": r[0], "reach_to_0": r[1], "unbalanced": r[2],
            "chaotic": r[0] == V and r[1] == V, "doubly_stochastic": r[2] == 0}
