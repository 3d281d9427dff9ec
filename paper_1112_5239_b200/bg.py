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


def _stream(stream):
    return ctypes.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)


def encrypt(chaotic: bool, N: torch.Tensor, r: torch.Tensor, m: torch.Tensor, S0: torch.Tensor | None = None,
            stream=None):
    """N, r: int64 [B]; m: uint8 [B, L]; S0: int32 [B] or None -> (c uint8 [B, L], y int64 [B])."""
    B, L = m.shape
    assert N.is_cuda and N.dtype == torch.int64 and N.numel() == B and r.numel() == B and m.dtype == torch.uint8
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
    c = c.contiguous()
    m = torch.empty_like(c)
    status = torch.empty(B, dtype=torch.int32, device=c.device)
    check(lib().prng_cbg_decrypt(int(chaotic), B, L, _p(p), _p(q), _p(S0), _p(c), _p(y), _p(m), _p(status),
                                 _stream(stream)), "prng_cbg_decrypt")
    return m, status
