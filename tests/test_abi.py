"""C-ABI library checks that need no GPU: the library loads, exports every
entry point include/ciprng.h declares, rejects bad configurations before
touching the device, and its division-free BBS squaring is exact."""
import ctypes
import subprocess

import pytest

import paper_1112_5239_b200 as P
from paper_1112_5239_b200 import _lib


def test_library_loads_and_exports_declared_symbols():
    L = P.lib()
    declared = P.declared_symbols()
    assert len(declared) >= 14
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in nm.splitlines() if " T " in ln}
    for name in declared:
        assert name in exported, name
        assert getattr(L, name) is not None


def test_version_string():
    assert b"sm_100a" in P.lib().prng_version()


def test_strerror_covers_all_statuses():
    for st in range(0, -8, -1):
        assert P.lib().prng_strerror(st) != b"unknown status"


def test_barrett_modsq_exhaustive():
    """Every modulus of the table, every y < M: barrett_sq and fbarrett_sq
    (host emulation of the FP32-quotient form) == y*y % M."""
    bad = ctypes.c_uint64(123)
    assert P.lib().prng_selftest_modsq(ctypes.byref(bad)) == 0
    assert bad.value == 0


def test_jump_ahead_selftest():
    """C1's single-stream split (csrc/v0_jump.cu): the host minimal
    polynomials of Listing 1's generators annihilate every basis vector, and
    jumps of J in {0 .. 299999} steps equal J plain steps from seeded states.
    xor64 and xorwow on 64-bit words have full-degree minimal polynomials
    (64, 320); Listing 1's xor128 on 64-bit words (shifts 11, 19, 8) has
    degree 253 < 256."""
    bad = ctypes.c_uint64(123)
    deg = (ctypes.c_uint32 * 3)()
    assert P.lib().prng_selftest_jump(ctypes.byref(bad), deg) == 0
    assert bad.value == 0
    assert list(deg) == [64, 253, 320]


def _create(seed, first, n_local, variant, comb_size=0, comb=None, paper_defaults=0, store_path=0):
    keep = None
    if comb is not None:
        keep = (ctypes.c_uint8 * len(comb))(*comb)
    cfg = _lib.PrngConfig(comb_size=comb_size, comb=ctypes.cast(keep, ctypes.c_void_p) if keep else None,
                          paper_defaults=paper_defaults, store_path=store_path)
    h = ctypes.c_void_p()
    rc = P.lib().prng_create_shard(seed, first, n_local, variant, ctypes.byref(cfg), ctypes.byref(h))
    if rc == 0:
        P.lib().prng_destroy(h)
    return rc


@pytest.mark.parametrize(
    "args",
    [
        dict(seed=0, first=0, n_local=32, variant=5),                     # unknown variant
        dict(seed=0, first=0, n_local=33, variant=3),                     # V3: incomplete group
        dict(seed=0, first=0, n_local=4, variant=4, comb_size=4),         # V4: defaults need C = 32
        dict(seed=0, first=0, n_local=0, variant=1),                      # no streams
        dict(seed=0, first=0, n_local=33, variant=1),                     # incomplete group
        dict(seed=0, first=16, n_local=32, variant=1),                    # misaligned shard
        dict(seed=0, first=0, n_local=4, variant=1, comb_size=3, comb=[0, 1, 2, 0, 1, 2]),  # C not 2^k
        dict(seed=0, first=0, n_local=4, variant=1, comb_size=4),         # defaults need C = 32
        dict(seed=0, first=0, n_local=4, variant=1, comb_size=4, comb=[0, 1, 2, 4, 0, 1, 2, 3]),  # entry >= C
        dict(seed=0, first=0, n_local=2, variant=0, paper_defaults=1),    # Q26
        dict(seed=0, first=0, n_local=32, variant=1, paper_defaults=1),
        dict(seed=0, first=0, n_local=32, variant=1, store_path=7),
    ],
)
def test_create_rejects_bad_config_without_device(args):
    assert _create(**args) == _lib.PRNG_EINVAL


def test_null_pointers_rejected():
    L = P.lib()
    assert L.prng_create(0, 32, 1, None) == _lib.PRNG_EINVAL
    assert L.prng_generate(None, 4, None, None) == _lib.PRNG_EINVAL
    assert L.prng_consume(None, 4, None, None) == _lib.PRNG_EINVAL
    assert L.prng_destroy(None) == 0


def test_sass_has_no_tensor_core_and_has_tma_store():
    """The V1 fast store kernel's tile path is a TMA bulk tensor store
    (UTMASTG / UBLKCP), and nothing here is a dense contraction (no UTC*MMA)."""
    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    sass = r.stdout
    assert "UTMASTG" in sass or "UBLKCP" in sass
    assert "UTCHMMA" not in sass and "HMMA" not in sass
    assert "SHFL.IDX" in sass


def test_next_rows_reject_bad_arguments_without_device():
    """NEXT-2..4 entry points validate before touching the device."""
    L = P.lib()
    E = _lib.PRNG_EINVAL
    assert L.prng_battery(None, 4, None, None) == E
    assert L.prng_cbg_encrypt(1, 4, 8, None, None, None, None, None, None, None) == E
    assert L.prng_cbg_decrypt(1, 4, 8, None, None, None, None, None, None, None, None) == E
    assert L.prng_cbg_encrypt(1, 0, 8, None, None, None, None, None, None, None) == 0  # no messages: no-op
    assert L.prng_alg1_generate(None, 8, 0, None, None, 4, 4, None, None) == E  # b = 0
    assert L.prng_alg1_generate(None, 33, 4, None, None, 4, 4, None, None) == E  # n > 32
    assert L.prng_alg1_generate(ctypes.c_void_p(16), 17, 4, None, None, 4, 4, None, None) == E  # table, n > 16
    assert L.prng_alg1_generate(None, 8, 4, None, None, 0, 4, None, None) == 0  # no streams: no-op
    assert L.prng_gamma_check(None, 0, None, None, None) == E
    assert L.prng_gamma_check(None, 17, ctypes.c_void_p(16), ctypes.c_void_p(16), None) == E


def test_python_binding_mirrors_abi_names():
    """The binding exposes every C-ABI entry point that takes work under its
    own name (marshalling only; no compute on import)."""
    compute = [s for s in P.declared_symbols() if s not in (
        "prng_strerror", "prng_last_cuda_error", "prng_selftest_modsq", "prng_selftest_modsq_gpu", "prng_selftest_jump",
        "prng_version")]
    missing = [s for s in compute if not callable(getattr(P, s, None))]
    assert not missing, missing


def _build_c_check(tmp_path):
    """tests/c_abi_check.c: include/ciprng.h as plain C99 (-pedantic), linked
    against libciprng.so (and the oracle for the GPU comparison)."""
    import os

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    import oracle

    oracle.build()
    libdir, odir = os.path.join(root, "paper_1112_5239_b200"), os.path.join(root, "oracle")
    exe = str(tmp_path / "c_abi_check")
    cmd = ["gcc", "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", "-I", os.path.join(root, "include"),
           os.path.join(root, "tests", "c_abi_check.c"), "-L", libdir, "-lciprng", "-L", odir, "-loracle",
           f"-Wl,-rpath,{libdir}", f"-Wl,-rpath,{odir}", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_abi_from_plain_c(tmp_path):
    """The boundary from plain C (no Python, no CUDA API, no GPU): the header
    compiles as C99, the library links, host self-tests and argument errors
    behave as include/ciprng.h states."""
    exe = _build_c_check(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "C ABI OK host" in r.stdout
