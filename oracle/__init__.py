"""CPU oracle for the chaotic-iteration PRNG hot path (arXiv 1112.5239).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_1112_5239_b200`` never imports it and
shares no code with it.

The arithmetic lives in ``ciprng_oracle.c`` (plain single-threaded C99, each
function citing the PAPER.md passage it follows).  This module is ctypes
marshalling only, plus numpy views of the oracle's per-stream structs.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ciprng_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

V0, V1, V2, V3, V4 = 0, 1, 2, 3, 4
# words (u32) per stream in the oracle's own structs (see ciprng_oracle.c)
STATE_WORDS = {V0: 24, V1: 6, V2: 18, V3: 4, V4: 24}


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, no vectorisation flags)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-std=c99", "-O2", "-fPIC", "-shared", "-Wall", "-Wextra", _SRC, "-o", _LIB]
        )
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        u64, u32, i32, vp = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_void_p
        L.orc_xor_step.argtypes, L.orc_xor_step.restype = [u64, u64], u64
        L.orc_xorshift32.argtypes, L.orc_xorshift32.restype = [vp], u32
        L.orc_xor64.argtypes, L.orc_xor64.restype = [vp], u64
        L.orc_xor128_64.argtypes, L.orc_xor128_64.restype = [vp], u64
        L.orc_xorwow_64.argtypes, L.orc_xorwow_64.restype = [vp, vp], u64
        L.orc_xor128_32.argtypes, L.orc_xor128_32.restype = [vp], u32
        L.orc_mix64.argtypes, L.orc_mix64.restype = [u64], u64
        L.orc_splitmix_word.argtypes, L.orc_splitmix_word.restype = [u64, u64, u32], u64
        L.orc_moduli.argtypes, L.orc_moduli.restype = [vp, i32], i32
        L.orc_bbs_step.argtypes, L.orc_bbs_step.restype = [u32, u32], u32
        L.orc_state_size.argtypes, L.orc_state_size.restype = [i32], ctypes.c_size_t
        L.orc_grid_init.argtypes, L.orc_grid_init.restype = [i32, u64, u64, u64, i32, vp], i32
        L.orc_init_from_words.argtypes, L.orc_init_from_words.restype = [i32, vp, vp], i32
        L.orc_grid_generate.argtypes = [i32, vp, u64, u32, vp, u64, vp]
        L.orc_grid_generate.restype = i32
        L.orc_stats_words.argtypes, L.orc_stats_words.restype = [vp, u64, u64, vp], i32
        L.orc_digest_words.argtypes, L.orc_digest_words.restype = [vp, u64, u64, u64], u64
        L.orc_battery_words.argtypes, L.orc_battery_words.restype = [vp, u64, u64, vp], i32
        L.orc_modmul.argtypes, L.orc_modmul.restype = [u64, u64, u64], u64
        L.orc_modpow.argtypes, L.orc_modpow.restype = [u64, u64, u64], u64
        L.orc_modinv.argtypes, L.orc_modinv.restype = [u64, u64, vp], i32
        L.orc_bg_unit_bits.argtypes, L.orc_bg_unit_bits.restype = [u64], u32
        L.orc_cbg_encrypt.argtypes = [i32, u64, u32, u64, u64, vp, vp, vp]
        L.orc_cbg_encrypt.restype = i32
        L.orc_cbg_decrypt.argtypes = [i32, u64, u64, u32, u64, vp, u64, vp]
        L.orc_cbg_decrypt.restype = i32
        L.orc_alg1_generate.argtypes = [vp, u32, u32, vp, vp, u64, u64, vp]
        L.orc_alg1_generate.restype = i32
        L.orc_gamma_check.argtypes, L.orc_gamma_check.restype = [vp, u32, vp], i32
        L.orc_gamma_reach.argtypes, L.orc_gamma_reach.restype = [vp, u32, vp], i32
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


# --------------------------------------------------------------------------
# scalar primitives
# --------------------------------------------------------------------------
def xor_step(x: int, s: int) -> int:
    return lib().orc_xor_step(x, s)


def xorshift32_seq(z: int, k: int) -> list[int]:
    st = np.array([z], dtype=np.uint32)
    return [lib().orc_xorshift32(_ptr(st)) for _ in range(k)]


def xor64_seq(a: int, k: int) -> list[int]:
    st = np.array([a], dtype=np.uint64)
    return [lib().orc_xor64(_ptr(st)) for _ in range(k)]


def xor128_64_seq(b, k: int) -> list[int]:
    st = np.array(b, dtype=np.uint64)
    return [lib().orc_xor128_64(_ptr(st)) for _ in range(k)]


def xorwow_64_seq(c, d: int, k: int) -> list[int]:
    st = np.array(c, dtype=np.uint64)
    dd = np.array([d], dtype=np.uint64)
    return [lib().orc_xorwow_64(_ptr(st), _ptr(dd)) for _ in range(k)]


def xor128_32_seq(b, k: int) -> list[int]:
    st = np.array(b, dtype=np.uint32)
    return [lib().orc_xor128_32(_ptr(st)) for _ in range(k)]


def mix64(z: int) -> int:
    return lib().orc_mix64(z)


def splitmix_word(seed: int, s: int, k: int) -> int:
    return lib().orc_splitmix_word(seed, s, k)


def moduli() -> list[int]:
    buf = np.zeros(256, dtype=np.uint32)
    n = lib().orc_moduli(_ptr(buf), 256)
    return [int(v) for v in buf[:n]]


def bbs_step(y: int, M: int) -> int:
    return lib().orc_bbs_step(y, M)


# --------------------------------------------------------------------------
# grid level
# --------------------------------------------------------------------------
class OracleError(RuntimeError):
    pass


def init_states(variant: int, seed: int, first_stream: int, n_local: int,
                paper_defaults: bool = False) -> np.ndarray:
    """Per-stream states as a (n_local, STATE_WORDS[variant]) uint32 array."""
    st = np.zeros((n_local, STATE_WORDS[variant]), dtype=np.uint32)
    rc = lib().orc_grid_init(variant, seed & (2**64 - 1), first_stream, n_local,
                             int(paper_defaults), _ptr(st))
    if rc != 0:
        raise OracleError(f"orc_grid_init rc={rc}")
    return st


def init_from_words(variant: int, words) -> np.ndarray:
    """One stream's state (STATE_WORDS[variant] uint32) from 16 injected seeder
    words w[k] (test hook: the Q11/Q21 word -> state mapping alone)."""
    w = np.zeros(16, dtype=np.uint64)
    w[: len(words)] = [int(v) & (2**64 - 1) for v in words]
    st = np.zeros((1, STATE_WORDS[variant]), dtype=np.uint32)
    rc = lib().orc_init_from_words(variant, _ptr(w), _ptr(st))
    if rc != 0:
        raise OracleError(f"orc_init_from_words rc={rc}")
    return st[0]


def generate(variant: int, states: np.ndarray, n: int, comb_size: int = 32,
             comb: np.ndarray | None = None) -> np.ndarray:
    """Advance `states` in place by one call of n rounds; returns (n_local, n) uint32."""
    assert states.dtype == np.uint32 and states.flags.c_contiguous
    n_local = states.shape[0]
    out = np.zeros((n_local, n), dtype=np.uint32)
    cb = None if comb is None else np.ascontiguousarray(comb, dtype=np.uint8)
    rc = lib().orc_grid_generate(variant, _ptr(states), n_local, comb_size, _ptr(cb), n, _ptr(out))
    if rc != 0:
        raise OracleError(f"orc_grid_generate rc={rc}")
    return out


def stats(words: np.ndarray, acc: np.ndarray | None = None) -> np.ndarray:
    """258 u64 consumer statistics of a (n_local, n) block of one call."""
    words = np.ascontiguousarray(words, dtype=np.uint32)
    acc = np.zeros(258, dtype=np.uint64) if acc is None else acc
    rc = lib().orc_stats_words(_ptr(words), words.shape[0], words.shape[1], _ptr(acc))
    if rc != 0:
        raise OracleError(f"orc_stats_words rc={rc}")
    return acc


N_BATTERY = 264


def battery(words: np.ndarray, acc: np.ndarray | None = None) -> np.ndarray:
    """264 u64 battery counts of a (n_local, n) block of one call (reading Q31)."""
    words = np.ascontiguousarray(words, dtype=np.uint32)
    acc = np.zeros(N_BATTERY, dtype=np.uint64) if acc is None else acc
    rc = lib().orc_battery_words(_ptr(words), words.shape[0], words.shape[1], _ptr(acc))
    if rc != 0:
        raise OracleError(f"orc_battery_words rc={rc}")
    return acc


# ------------------------------------------------- Blum-Goldwasser (NEXT-3)
def modpow(a: int, e: int, m: int) -> int:
    return lib().orc_modpow(a, e, m)


def modinv(a: int, m: int) -> int:
    out = np.zeros(1, np.uint64)
    if lib().orc_modinv(a, m, _ptr(out)) != 0:
        raise OracleError("not invertible")
    return int(out[0])


def bg_unit_bits(N: int) -> int:
    return lib().orc_bg_unit_bits(N)


def cbg_encrypt(chaotic: bool, N: int, S0: int, r: int, m) -> tuple[np.ndarray, int]:
    """(c units, y); classic BG when chaotic is False (units = bits)."""
    m = np.ascontiguousarray(m, dtype=np.uint8)
    c = np.zeros_like(m)
    y = np.zeros(1, np.uint64)
    if lib().orc_cbg_encrypt(int(chaotic), N, S0, r, m.size, _ptr(m), _ptr(c), _ptr(y)) != 0:
        raise OracleError("cbg_encrypt: invalid key or r")
    return c, int(y[0])


def cbg_decrypt(chaotic: bool, p: int, q: int, S0: int, c, y: int) -> np.ndarray:
    c = np.ascontiguousarray(c, dtype=np.uint8)
    m = np.zeros_like(c)
    if lib().orc_cbg_decrypt(int(chaotic), p, q, S0, c.size, _ptr(c), y, _ptr(m)) != 0:
        raise OracleError("cbg_decrypt: invalid key or ciphertext")
    return m


# ------------------------------------------------ Algorithm 1 + Gamma(f) (NEXT-4)
def alg1_generate(f, n: int, b: int, z: np.ndarray, x: np.ndarray, n_out: int) -> np.ndarray:
    """Algorithm 1, n_out calls per stream; z, x (uint32 [S]) advance in place."""
    ft = None if f is None else np.ascontiguousarray(f, dtype=np.uint32)
    S = z.size
    out = np.zeros((S, n_out), dtype=np.uint32)
    rc = lib().orc_alg1_generate(_ptr(ft), n, b, _ptr(z), _ptr(x), S, n_out, _ptr(out))
    if rc != 0:
        raise OracleError("alg1_generate")
    return out


def gamma_check(f, n: int) -> dict:
    ft = None if f is None else np.ascontiguousarray(f, dtype=np.uint32)
    rep = np.zeros(3, np.uint64)
    if lib().orc_gamma_check(_ptr(ft), n, _ptr(rep)) != 0:
        raise OracleError("gamma_check")
    return {"scc": int(rep[0]), "doubly_stochastic": bool(rep[1]), "unbalanced": int(rep[2])}


def gamma_reach(f, n: int) -> np.ndarray:
    """[reachable from 0, reaching 0, unbalanced vertices] (orc_gamma_reach)."""
    ft = None if f is None else np.ascontiguousarray(f, dtype=np.uint32)
    rep = np.zeros(3, np.uint64)
    if lib().orc_gamma_reach(_ptr(ft), n, _ptr(rep)) != 0:
        raise OracleError("gamma_reach")
    return rep


def digest(words: np.ndarray, first_stream: int = 0) -> int:
    words = np.ascontiguousarray(words, dtype=np.uint32)
    return lib().orc_digest_words(_ptr(words), first_stream, words.shape[0], words.shape[1])


def state_planes(variant: int, states: np.ndarray) -> np.ndarray:
    """The oracle's per-stream structs viewed as the C-ABI's SoA u32 planes
    (include/ciprng.h, "State layout"): plane k holds word k of every stream.
    V0 drops the struct's trailing pad word."""
    nplanes = {V0: 23, V1: 6, V2: 18, V3: 4, V4: 24}[variant]
    return np.ascontiguousarray(states[:, :nplanes].T)


def states_from_planes(variant: int, planes: np.ndarray) -> np.ndarray:
    n_local = planes.shape[1]
    st = np.zeros((n_local, STATE_WORDS[variant]), dtype=np.uint32)
    st[:, : planes.shape[0]] = planes.T
    return st
