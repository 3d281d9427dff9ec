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


def _vec(t: torch.Tensor, numel: int, dev, name: str) -> None:
    """A device vector argument: contiguous int32 [numel] on `dev` (the kernels
    index it up to numel - 1, so a shorter tensor would be read out of bounds)."""
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.device == dev and t.dtype == torch.int32
            and t.numel() == numel and t.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous int32 [{numel}] CUDA tensor on {dev}")


def _table(f: torch.Tensor | None, n: int, dev) -> None:
    """f as a table: int32 [2^n] on `dev` (f_single reads f[x] for every x < 2^n)."""
    if f is not None:
        _vec(f, 1 << n, dev, f"f (table of 2^{n} entries)")


def alg1_generate(n: int, b: int, z: torch.Tensor, x: torch.Tensor, n_out: int, f: torch.Tensor | None = None,
                  stream=None) -> torch.Tensor:
    """z, x: int32 CUDA [S] (u32 bits), advanced in place -> int32 [S, n_out]."""
    if not isinstance(z, torch.Tensor) or not z.is_cuda:
        raise ValueError("z must be an int32 CUDA tensor")
    S = z.numel()
    _vec(z, S, z.device, "z")
    _vec(x, S, z.device, "x")
    _table(f, n, z.device)
    out = torch.empty((S, n_out), dtype=torch.int32, device=z.device)
    check(lib().prng_alg1_generate(_p(f), n, b, _p(z), _p(x), S, n_out, _p(out), _stream(stream)),
          "prng_alg1_generate")
    return out


def gamma_check(n: int, f: torch.Tensor | None = None, device="cuda", stream=None) -> dict:
    if f is not None:
        device = f.device
    device = torch.device(device)
    if device.type == "cuda" and device.index is None:
        device = torch.device("cuda", torch.cuda.current_device())
    _table(f, n, device)
    scratch = torch.empty(1 << n, dtype=torch.uint8, device=device)
    rep = torch.zeros(3, dtype=torch.int64, device=device)
    check(lib().prng_gamma_check(_p(f), n, _p(scratch), _p(rep), _stream(stream)), "prng_gamma_check")
    r = rep.cpu().tolist()
    V = 1 << n
    return {"reach_from_0": r[0], "reach_to_0": r[1], "unbalanced": r[2],
            "chaotic": r[0] == V and r[1] == V, "doubly_stochastic": r[2] == 0}
