"""Seeded synthetic workloads shared by tests/, bench.py and smoke().

This module holds NO arithmetic of the method: only the seeds, the shapes of
BASELINE.json's configs and numpy-seeded generators for test inputs (custom
combination tables, injected states).  Both the oracle side and the CUDA side
receive what it produces as plain inputs.

Shapes follow the paper's workloads: 30k-5M threads with tens to hundreds of
numbers each -- see DESIGN.md s5 for the recipe.
"""
from __future__ import annotations

import numpy as np

V0, V1, V2, V3, V4 = 0, 1, 2, 3, 4
VARIANT_NAMES = {V0: "v0_xorlike3", V1: "v1_xor128_comb", V2: "v2_bbs_comb", V3: "v3_xor64_comb",
                 V4: "v4_xorlike3_comb"}

# fixed seed list; timing uses the first
SEEDS = [0x0123456789ABCDEF, 0, 0xFFFFFFFFFFFFFFFF]

# BASELINE.json configs[0..4]
CONFIGS = {
    "C1": dict(variant=V0, n_streams=1, n=10**6, paper_defaults=True, calls=1),
    "C2": dict(variant=V1, n_streams=2**20, n=128, calls=1),
    "C3": dict(variant=V2, n_streams=2**20, n=64, calls=1),
    "C4": dict(variant=V1, n_streams=2**23, n=256, calls=466),
    "C5": dict(variant=V1, n_streams=2**23, n=1024, calls=16, mode="consume"),
}


def rng(tag: int) -> np.random.Generator:
    return np.random.default_rng(0xC1A05 + tag)


def random_comb(gen: np.random.Generator, comb_size: int, n_tables: int) -> np.ndarray:
    """n_tables combination arrays of size comb_size: each a random
    permutation of 0..C-1 ("a combination array that contains the indexes of
    all threads").  Returned flat, table-major, uint8."""
    return np.concatenate([gen.permutation(comb_size) for _ in range(n_tables)]).astype(np.uint8)


def random_words(gen: np.random.Generator, shape) -> np.ndarray:
    return gen.integers(0, 2**32, size=shape, dtype=np.uint64).astype(np.uint32)


# ---------------------------------------------------- Blum-Goldwasser inputs
_MR_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def _is_prime(v: int) -> bool:
    """Deterministic Miller-Rabin for v < 3.3e24 (key generation input only)."""
    if v < 2:
        return False
    for p in _MR_BASES:
        if v % p == 0:
            return v == p
    d, s = v - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in _MR_BASES:
        x = pow(a, d, v)
        if x in (1, v - 1):
            continue
        for _ in range(s - 1):
            x = x * x % v
            if x == v - 1:
                break
        else:
            return False
    return True


def blum_prime(gen: np.random.Generator, bits: int) -> int:
    """A random prime p = 3 (mod 4) with the given bit length."""
    while True:
        v = int(gen.integers(2 ** (bits - 1), 2**bits)) | 3
        if _is_prime(v):
            return v


def bg_keys(gen: np.random.Generator, count: int, bits: int):
    """count key pairs (p, q, N = p q) with p != q Blum primes of `bits` bits."""
    out = []
    while len(out) < count:
        p, q = blum_prime(gen, bits), blum_prime(gen, bits)
        if p != q:
            out.append((p, q, p * q))
    return out
