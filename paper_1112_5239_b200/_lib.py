"""ctypes binding of libciprng.so (include/ciprng.h).  Argument marshalling
only: every step of the hot path runs in the library's CUDA kernels.  There is
no fallback: if the shared library is missing the import fails loudly."""
from __future__ import annotations

import ctypes
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libciprng.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "ciprng.h")

PRNG_OK, PRNG_EINVAL, PRNG_ENOMEM, PRNG_ECUDA, PRNG_EALIGN, PRNG_ESIZE, PRNG_ESTATE, PRNG_EIO = \
    0, -1, -2, -3, -4, -5, -6, -7
STORE_AUTO, STORE_DIRECT, STORE_TMA = 0, 1, 2
EMIT_FORMATS = {"raw-le32": 0, "hex": 1, "bits": 2}


class PrngConfig(ctypes.Structure):
    _fields_ = [
        ("comb_size", ctypes.c_uint32),
        ("comb", ctypes.c_void_p),
        ("paper_defaults", ctypes.c_int32),
        ("store_path", ctypes.c_int32),
    ]


class PrngInfo(ctypes.Structure):
    _fields_ = [
        ("variant", ctypes.c_int32),
        ("comb_size", ctypes.c_uint32),
        ("seed", ctypes.c_uint64),
        ("first_stream", ctypes.c_uint64),
        ("n_local", ctypes.c_uint64),
        ("state_words", ctypes.c_uint32),
        ("device", ctypes.c_int32),
        ("store_path", ctypes.c_int32),
        ("kernel_launches", ctypes.c_uint32),
    ]


class PrngError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        msg = lib().prng_strerror(status).decode()
        if status == PRNG_ECUDA:
            msg += ": " + lib().prng_last_cuda_error().decode()
        super().__init__(f"{what}: {msg} (status {status})")


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} not built: run `python __graft_entry__.py build` (nvcc, sm_100a). "
                "There is no CPU fallback."
            )
        L = ctypes.CDLL(LIB_PATH)
        u64, u32, i32, vp, sz = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t
        H = ctypes.POINTER(ctypes.c_void_p)
        sig = {
            "prng_create": ([u64, u64, i32, H], i32),
            "prng_create_shard": ([u64, u64, u64, i32, ctypes.POINTER(PrngConfig), H], i32),
            "prng_destroy": ([vp], i32),
            "prng_generate": ([vp, u64, vp, vp], i32),
            "prng_generate_host": ([vp, u64, vp, vp], i32),
            "prng_emit": ([vp, u64, i32, i32, ctypes.POINTER(u64), vp], i32),
            "prng_consume": ([vp, u64, vp, vp], i32),
            "prng_battery": ([vp, u64, vp, vp], i32),
            "prng_cbg_encrypt": ([i32, u64, u64, vp, vp, vp, vp, vp, vp, vp], i32),
            "prng_cbg_decrypt": ([i32, u64, u64, vp, vp, vp, vp, vp, vp, vp, vp], i32),
            "prng_alg1_generate": ([vp, u32, u32, vp, vp, u64, u64, vp, vp], i32),
            "prng_gamma_check": ([vp, u32, vp, vp, vp], i32),
            "prng_digest": ([vp, u64, u64, u64, vp, vp], i32),
            "prng_get_info": ([vp, ctypes.POINTER(PrngInfo)], i32),
            "prng_get_state": ([vp, vp, sz], i32),
            "prng_set_state": ([vp, vp, sz], i32),
            "prng_strerror": ([i32], ctypes.c_char_p),
            "prng_last_cuda_error": ([], ctypes.c_char_p),
            "prng_selftest_modsq": ([ctypes.POINTER(u64)], i32),
            "prng_selftest_modsq_gpu": ([ctypes.POINTER(u64)], i32),
            "prng_selftest_jump": ([ctypes.POINTER(u64), ctypes.POINTER(u32)], i32),
            "prng_version": ([], ctypes.c_char_p),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes, f.restype = args, res
        _lib = L
    return _lib


def check(status: int, what: str) -> None:
    if status != PRNG_OK:
        raise PrngError(status, what)


def declared_symbols() -> list[str]:
    """Entry points declared in include/ciprng.h."""
    with open(HEADER) as fh:
        txt = fh.read()
    return sorted(set(re.findall(r"CIPRNG_API\s+[\w\s\*]+?\b(prng_\w+)\s*\(", txt)))
