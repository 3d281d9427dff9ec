"""B200-native chaotic-iteration PRNG (arXiv 1112.5239) -- Python binding.

``ChaoticPRNG`` wraps one C-ABI handle (include/ciprng.h).  PyTorch supplies
device memory, streams and (for multi-GPU) the process group; every step of
the hot path -- seeding, strategy generation, neighbour combination, the
chaotic-iteration update, stores or the fused consumer -- runs in this
package's sm_100a kernels (csrc/).  Importing works on a CPU-only host (the
library loads), but every compute call needs a CUDA device: there is no CPU
fallback.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from ._lib import (  # noqa: F401
    EMIT_FORMATS,
    STORE_AUTO,
    STORE_DIRECT,
    STORE_TMA,
    PrngConfig,
    PrngError,
    PrngInfo,
    check,
    declared_symbols,
    lib,
)

V0, V1, V2, V3, V4 = 0, 1, 2, 3, 4
STATE_WORDS = {V0: 23, V1: 6, V2: 18, V3: 4, V4: 24}
N_STATS = 258
N_BATTERY = 264

__all__ = ["ChaoticPRNG", "digest", "V0", "V1", "V2", "V3", "V4", "STATE_WORDS", "N_STATS", "N_BATTERY", "lib",
           "PrngError"]


def _require(cond: bool, msg: str) -> None:
    """Argument validation that survives ``python -O`` (unlike assert)."""
    if not cond:
        raise ValueError(msg)


def _stream_handle(stream) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


class ChaoticPRNG:
    """Per-stream chaotic-iteration generators for global streams
    [first, first + n_local) of the stream space of ``seed``.

    variant: V0 (Listing 1 / Alg. 3), V1 (Alg. 4), V2 (Alg. 5, BBS), V3 (Alg. 4 with
    the xor64 source of the paper's optimized kernels), V4 (Alg. 4 with Listing
    1's three-generator fold as the source).
    comb_size / comb: combination arrays (None = default C = 32 tables).
    """

    def __init__(self, seed: int, n_streams: int, variant: int = V1, *, shard: tuple[int, int] | None = None,
                 comb_size: int | None = None, comb=None, paper_defaults: bool = False,
                 store_path: int = STORE_AUTO, device=None):
        if not torch.cuda.is_available():
            raise RuntimeError("ChaoticPRNG needs a CUDA device (sm_100a); there is no CPU fallback")
        self.variant = variant
        self.seed = seed & (2**64 - 1)
        first, n_local = shard if shard is not None else (0, n_streams)
        self.first, self.n_local, self.n_streams = first, n_local, n_streams
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else torch.device(device).index)
        self._comb = None if comb is None else np.ascontiguousarray(comb, dtype=np.uint8)
        if self._comb is not None:
            # prng_create_shard reads ntab * C bytes from this host pointer
            ntab = 16 if variant == V2 else 2
            _require(self._comb.size == ntab * (comb_size or 32),
                     f"comb must hold {ntab} x comb_size = {ntab * (comb_size or 32)} entries, got {self._comb.size}")
        cfg = PrngConfig(
            comb_size=comb_size or 0,
            comb=None if self._comb is None else self._comb.ctypes.data,
            paper_defaults=int(paper_defaults),
            store_path=store_path,
        )
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            check(lib().prng_create_shard(self.seed, first, n_local, variant, ctypes.byref(cfg), ctypes.byref(h)),
                  "prng_create_shard")
        self._h = h

    # ----------------------------------------------------------------- hot path
    def generate(self, n: int, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """One call of n rounds; returns int32 [n_local, n] (bit pattern = u32)."""
        if out is None:
            out = torch.empty((self.n_local, n), dtype=torch.int32, device=self.device)
        _require(out.is_cuda and out.device == self.device, f"out must live on {self.device}")
        _require(out.is_contiguous() and out.element_size() == 4 and out.numel() >= self.n_local * n,
                 f"out must be a contiguous 4-byte tensor of >= {self.n_local} x {n} elements")
        check(lib().prng_generate(self._h, n, ctypes.c_void_p(out.data_ptr()), _stream_handle(stream)),
              "prng_generate")
        return out

    def generate_host(self, n: int, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """Same words into a (pinned) host tensor, overlapping D2H with generation."""
        if out is None:
            out = torch.empty((self.n_local, n), dtype=torch.int32, pin_memory=True)
        _require(not out.is_cuda and out.is_contiguous() and out.element_size() == 4
                 and out.numel() >= self.n_local * n,
                 f"out must be a contiguous 4-byte host tensor of >= {self.n_local} x {n} elements")
        check(lib().prng_generate_host(self._h, n, ctypes.c_void_p(out.data_ptr()), _stream_handle(stream)),
              "prng_generate_host")
        return out

    def emit(self, n: int, sink, format: str = "raw-le32", stream=None) -> int:
        """One call of n rounds serialised to `sink` (an int file descriptor,
        a path, or a file object with fileno(); include/ciprng.h prng_emit):
        format "raw-le32", "hex" or "bits".  Returns the bytes
        written; the words are prng_generate's, in its order."""
        _require(format in EMIT_FORMATS, f"format must be one of {sorted(EMIT_FORMATS)}")
        close = False
        if isinstance(sink, int):
            fd = sink
        elif isinstance(sink, (str, bytes)) or hasattr(sink, "__fspath__"):
            fd = os.open(sink, os.O_WRONLY | os.O_CREAT | os.O_TRUNC, 0o644)
            close = True
        else:
            sink.flush()
            fd = sink.fileno()
        written = ctypes.c_uint64(0)
        try:
            check(lib().prng_emit(self._h, n, fd, EMIT_FORMATS[format], ctypes.byref(written),
                                  _stream_handle(stream)), "prng_emit")
        finally:
            if close:
                os.close(fd)
        return written.value

    def consume(self, n: int, stats: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """Fused consumer: adds {inside, pairs, hist[256]} into int64 [258] (u64 bits)."""
        if stats is None:
            stats = torch.zeros(N_STATS, dtype=torch.int64, device=self.device)
        _require(stats.is_cuda and stats.device == self.device and stats.numel() == N_STATS
                 and stats.dtype == torch.int64 and stats.is_contiguous(),
                 f"stats must be a contiguous int64 [{N_STATS}] tensor on {self.device}")
        check(lib().prng_consume(self._h, n, ctypes.c_void_p(stats.data_ptr()), _stream_handle(stream)),
              "prng_consume")
        return stats

    def battery(self, n: int, stats: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """Statistical-battery counts (include/ciprng.h prng_battery): adds into
        int64 [264] (u64 bits).  P-values: ``battery.pvalues``."""
        if stats is None:
            stats = torch.zeros(N_BATTERY, dtype=torch.int64, device=self.device)
        _require(stats.is_cuda and stats.device == self.device and stats.numel() == N_BATTERY
                 and stats.dtype == torch.int64 and stats.is_contiguous(),
                 f"stats must be a contiguous int64 [{N_BATTERY}] tensor on {self.device}")
        check(lib().prng_battery(self._h, n, ctypes.c_void_p(stats.data_ptr()), _stream_handle(stream)),
              "prng_battery")
        return stats

    # ------------------------------------------------------------ introspection
    def info(self) -> PrngInfo:
        inf = PrngInfo()
        check(lib().prng_get_info(self._h, ctypes.byref(inf)), "prng_get_info")
        return inf

    def get_state(self) -> np.ndarray:
        """SoA state planes, uint32 [state_words, n_local] (include/ciprng.h)."""
        buf = np.zeros((STATE_WORDS[self.variant], self.n_local), dtype=np.uint32)
        check(lib().prng_get_state(self._h, ctypes.c_void_p(buf.ctypes.data), buf.nbytes), "prng_get_state")
        return buf

    def set_state(self, planes: np.ndarray) -> None:
        """Checkpoint resume: SoA planes uint32 [state_words, n_local]; the
        library rejects (PrngError, PRNG_ESTATE) a wrong size or invalid content."""
        buf = np.ascontiguousarray(planes, dtype=np.uint32)
        check(lib().prng_set_state(self._h, ctypes.c_void_p(buf.ctypes.data), buf.nbytes), "prng_set_state")

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().prng_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def digest(out: torch.Tensor, first_stream: int = 0, acc: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Position-aware verification digest of a [n_local, n] output block (Q28)."""
    _require(out.is_cuda and out.dim() == 2 and out.is_contiguous() and out.element_size() == 4,
             "out must be a contiguous 2-D 4-byte CUDA tensor")
    n_local, n = out.shape
    if acc is None:
        acc = torch.zeros(1, dtype=torch.int64, device=out.device)
    check(lib().prng_digest(ctypes.c_void_p(out.data_ptr()), first_stream, n_local, n,
                            ctypes.c_void_p(acc.data_ptr()), _stream_handle(stream)), "prng_digest")
    return acc


def as_u32(t: torch.Tensor) -> np.ndarray:
    """Copy a device/host int32 tensor to a numpy uint32 array (bit-exact)."""
    return t.detach().cpu().numpy().view(np.uint32)


def as_u64(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy().view(np.uint64)


# ---------------------------------------------------------------------------
# The C-ABI entry points under their own names (include/ciprng.h), for users
# who think in the C interface; each is marshalling over the calls above.
# ---------------------------------------------------------------------------
def prng_create(seed: int, n_streams: int, variant: int = V1, **kw) -> ChaoticPRNG:
    """prng_create(seed, n_streams, variant) -> handle (north_star signature)."""
    return ChaoticPRNG(seed, n_streams, variant, **kw)


def prng_create_shard(seed: int, first_stream: int, n_local: int, variant: int = V1, **kw) -> ChaoticPRNG:
    return ChaoticPRNG(seed, first_stream + n_local, variant, shard=(first_stream, n_local), **kw)


def prng_generate(h: ChaoticPRNG, n_per_stream: int, out=None, stream=None):
    return h.generate(n_per_stream, out=out, stream=stream)


def prng_generate_host(h: ChaoticPRNG, n_per_stream: int, out=None, stream=None):
    return h.generate_host(n_per_stream, out=out, stream=stream)


def prng_emit(h: ChaoticPRNG, n_per_stream: int, sink, format: str = "raw-le32", stream=None) -> int:
    return h.emit(n_per_stream, sink, format, stream=stream)


def prng_consume(h: ChaoticPRNG, n_per_stream: int, stats=None, stream=None):
    return h.consume(n_per_stream, stats, stream=stream)


def prng_battery(h: ChaoticPRNG, n_per_stream: int, stats=None, stream=None):
    return h.battery(n_per_stream, stats, stream=stream)


def prng_digest(out, first_stream: int = 0, acc=None, stream=None):
    return digest(out, first_stream, acc, stream)


def prng_get_state(h: ChaoticPRNG):
    return h.get_state()


def prng_set_state(h: ChaoticPRNG, planes) -> None:
    h.set_state(planes)


def prng_get_info(h: ChaoticPRNG):
    return h.info()


def prng_destroy(h: ChaoticPRNG) -> None:
    h.close()


def prng_cbg_encrypt(chaotic, N, r, m, S0=None, stream=None):
    from . import bg

    return bg.encrypt(chaotic, N, r, m, S0, stream)


def prng_cbg_decrypt(chaotic, p, q, c, y, S0=None, stream=None):
    from . import bg

    return bg.decrypt(chaotic, p, q, c, y, S0, stream)


def prng_alg1_generate(n, b, z, x, n_out, f=None, stream=None):
    from . import chaos

    return chaos.alg1_generate(n, b, z, x, n_out, f, stream)


def prng_gamma_check(n, f=None, stream=None):
    from . import chaos

    return chaos.gamma_check(n, f, stream=stream)
