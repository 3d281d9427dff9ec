"""Blum-Goldwasser and the paper's chaotic variant (
PAPER.md P:1327-1386), batched on the GPU: thin marshalling over the C-ABI
``prng_cbg_encrypt`` / ``prng_cbg_decrypt`` (include/ciprng.h).  Tensors are
CUDA tensors; 64-bit values travel as int64 bit patterns."""
from __future__ import annotations

import ctypes

import torch

from ._lib import check, lib


def _p(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _vec(t: torch.Tensor | None, B: int, dtype, dev, name: str) -> None:
    """A per-message vector argument: contiguous, [B], of `dtype`, on `dev` (None allowed only for S0)."""
    if t is None:
        return
    if not (t.is_cuda and t.device == dev and t.dtype == dtype and t.numel() == B and t.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous {dtype} [{B}] tensor on {dev}")


def _stream(stream):
    return ctypes.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)


def encrypt(chaotic: bool, N: torch.Tensor, r: torch.Tensor, m: torch.Tensor, S0: torch.Tensor | None = None,
            stream=None):
    """N, r: int64 [B]; m: uint8 [B, L]; S0: int32 [B] or None -> (c uint8 [B, L], y int64 [B])."""
    B, L = m.shape
    if not (m.is_cuda and m.dtype == torch.uint8):
        raise ValueError("m must be a uint8 [B, L] CUDA tensor")
    for t, dt, name in ((N, torch.int64, "N"), (r, torch.int64, "r"), (S0, torch.int32, "S0")):
        _vec(t, B, dt, m.device, name)
    m = m.contiguous()
    c = torch.empty_like(m)
    y = torch.empty(B, dtype=torch.int64, device=m.device)
    check(lib().prng_cbg_encrypt(int(chaotic), B, L, _p(N), _p(S0), _p(r), _p(m), _p(c), _p(y), _stream(stream)),
          "prng_cbg_encrypt")
    return c, y


def decrypt(chaotic: bool, p: torch.Tensor, q: torch.Tensor, c: torch.Tensor, y: torch.Tensor,
            S0: torch.Tensor | None = None, stream=None):
    """-> (m uint8 [B, L], status int32 [B]: 0 ok, 1 invalid key / y)."""
    B, L = c.shape
    if not (c.is_cuda and c.dtype == torch.uint8):
        raise ValueError("c must be a uint8 [B, L] CUDA tensor")
    for t, dt, name in ((p, torch.int64, "p"), (q, torch.int64, "q"), (y, torch.int64, "y"), (S0, torch.int32, "S0")):
        _vec(t, B, dt, c.device, name)
    c = c.contiguous()
    m = torch.empty_like(c)
    status = torch.empty(B, dtype=torch.int32, device=c.device)
    check(lib().prng_cbg_decrypt(int(chaotic), B, L, _p(p), _p(q), _p(S0), _p(c), _p(y), _p(m), _p(status),
                                 _stream(stream)), "prng_cbg_decrypt")
    return m, status
