"""GPU parity: the CUDA path through the C-ABI against the CPU oracle, word
for word (bit-exact: the method is integer-only, so exactly one output is
correct under the DESIGN.md readings).  Sizes span several warps/tiles and a
ragged tail; edge cases: n = 0, n not a multiple of 4, incomplete last tile,
custom combination arrays, multi-call state carry, V2 per-call selection and
rotation, shards, host-buffer path, misaligned outputs."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_1112_5239_b200 as P
import workloads as W
from tests.gpu_helpers import first_mismatch, gpu_run, oracle_run

pytestmark = pytest.mark.gpu

SEEDS = W.SEEDS
NS = [0, 1, 3, 4, 5, 127, 128, 1000]


def _check(variant, seed, S, ns, **kw):
    comb_size = kw.pop("comb_size", None)
    comb = kw.pop("comb", None)
    store_path = kw.pop("store_path", P.STORE_AUTO)
    first = kw.pop("first", 0)
    paper_defaults = kw.pop("paper_defaults", False)
    outs, planes, info = gpu_run(variant, seed, S, ns, first=first, comb_size=comb_size, comb=comb,
                                 paper_defaults=paper_defaults, store_path=store_path, **kw)
    ro, rplanes = oracle_run(variant, seed, S, ns, first=first, comb_size=comb_size or 32, comb=comb,
                             paper_defaults=paper_defaults)
    for k, (a, b) in enumerate(zip(outs, ro)):
        assert np.array_equal(a, b), f"call {k} (n={ns[k]}): {first_mismatch(a, b)}"
    assert np.array_equal(planes, rplanes), f"state: {first_mismatch(planes, rplanes)}"
    return info


# ------------------------------------------------------------------------ V1
@pytest.mark.parametrize("seed", SEEDS)
@pytest.mark.parametrize("S", [32, 64, 96, 1024, 16384])
@pytest.mark.parametrize("store_path", [P.STORE_DIRECT, P.STORE_TMA])
def test_v1_default_tables(seed, S, store_path):
    info = _check(W.V1, seed, S, NS, store_path=store_path)
    assert info.kernel_launches == 1


@pytest.mark.parametrize("C", [1, 2, 4, 8, 32])
def test_v1_custom_tables(C):
    gen = W.rng(100 + C)
    comb = W.random_comb(gen, C, 2)
    for S in (C * 3 if C < 32 else 64, 1024):
        _check(W.V1, SEEDS[0], S, [5, 128, 3], comb_size=C, comb=comb)


@pytest.mark.parametrize("S", [96, 4096 + 32, 65536])
def test_v1_default_shape_by_n(S):
    """The default V1 store picks its box shape by n (2-D 32-round boxes for
    n < 192, 3-D 64-round band boxes for n >= 192, n % 32 == 0; api.cu):
    calls alternating between the two shapes, incl. a partial last band
    (n = 224), continue every stream bit-exactly."""
    _check(W.V1, SEEDS[1], S, [192, 128, 256, 224, 1024, 36, 320], store_path=P.STORE_TMA)


def test_v1_spec_tiny_tables():
    """T=4, c=2, comb1=[0,1], comb2=[1,0]."""
    _check(W.V1, 12345, 4, [1, 2, 7], comb_size=2, comb=np.array([0, 1, 1, 0], np.uint8))


def test_v1_shard_equals_slice():
    S = 2048
    whole, _, _ = gpu_run(W.V1, SEEDS[0], S, [64])
    lo, _, _ = gpu_run(W.V1, SEEDS[0], S // 2, [64], first=0)
    hi, _, _ = gpu_run(W.V1, SEEDS[0], S // 2, [64], first=S // 2)
    assert np.array_equal(np.concatenate([lo[0], hi[0]]), whole[0])


def test_v1_split_invariance_gpu():
    a, _, _ = gpu_run(W.V1, 7, 256, [100])
    b, _, _ = gpu_run(W.V1, 7, 256, [36, 64])
    assert np.array_equal(a[0], np.concatenate(b, axis=1))


def test_v1_misaligned_output_falls_back():
    """Output pointer 4 bytes off 16-byte alignment: AUTO/DIRECT fall back to
    scalar stores and stay exact; explicit TMA reports PRNG_EALIGN."""
    _check(W.V1, 3, 128, [8, 12], out_offset_words=1)
    _check(W.V1, 3, 128, [8], out_offset_words=1, store_path=P.STORE_DIRECT)
    with pytest.raises(P.PrngError) as ei:
        gpu_run(W.V1, 3, 128, [8], out_offset_words=1, store_path=P.STORE_TMA)
    assert ei.value.status == -4


@pytest.mark.parametrize("variant", [W.V0, W.V1, W.V2, W.V3, W.V4])
def test_zero_rounds_is_a_noop(variant):
    """n_per_stream == 0 is a no-op for every variant (include/ciprng.h): no
    launch, state untouched -- for V2 in particular no per-call rotation
    (reading Q19) -- so a 0-round call between two calls changes nothing;
    consume(0) adds nothing."""
    info = _check(variant, SEEDS[0], 96, [5, 0, 8])
    g = P.ChaoticPRNG(SEEDS[0], 96, variant)
    before = g.get_state()
    stats = g.consume(0)
    assert g.info().kernel_launches == 0
    assert not P.as_u64(stats).any() and np.array_equal(g.get_state(), before)
    g.close()
    assert info is not None


def test_size_overflow_rejected_before_launch():
    """n * n_local * 4 beyond size_t is PRNG_ESIZE, returned before any launch
    (the pointer is never dereferenced); the state is untouched."""
    import ctypes

    g = P.ChaoticPRNG(SEEDS[0], 64, W.V1)
    before = g.get_state()
    dummy = torch.empty(4, dtype=torch.int32, device="cuda")
    st = P.lib().prng_generate(g._h, 2**62, ctypes.c_void_p(dummy.data_ptr()), ctypes.c_void_p(0))
    assert st == P._lib.PRNG_ESIZE and g.info().kernel_launches == 0
    assert np.array_equal(g.get_state(), before)
    g.close()


def test_binding_rejects_bad_buffers():
    """The binding validates buffers with exceptions (not asserts, which
    python -O strips): wrong dtype size, too small, host vs device, stats
    shape; the handle's state is untouched by a rejected call."""
    g = P.ChaoticPRNG(SEEDS[0], 64, W.V1)
    before = g.get_state()
    with pytest.raises(ValueError):
        g.generate(8, out=torch.empty((64, 8), dtype=torch.int64, device="cuda"))
    with pytest.raises(ValueError):
        g.generate(8, out=torch.empty((64, 7), dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError):
        g.generate(8, out=torch.empty((64, 8), dtype=torch.int32))
    with pytest.raises(ValueError):
        g.generate_host(8, out=torch.empty((64, 8), dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError):
        g.consume(8, torch.zeros(257, dtype=torch.int64, device="cuda"))
    with pytest.raises(ValueError):
        g.battery(8, torch.zeros(P.N_BATTERY, dtype=torch.int32, device="cuda"))
    assert np.array_equal(g.get_state(), before)
    g.close()


def test_v0_generate_host_single_stream_jump():
    """generate_host on a one-stream V0 handle (C1's shape) takes the jump
    path inside the host pipeline and equals generate word for word, over
    two calls (state carried)."""
    g1 = P.ChaoticPRNG(0, 1, W.V0, paper_defaults=True)
    g2 = P.ChaoticPRNG(0, 1, W.V0, paper_defaults=True)
    for n in (10**6, 5003):
        dev = P.as_u32(g1.generate(n))
        host = g2.generate_host(n).numpy().view(np.uint32)
        assert np.array_equal(dev, host)
    assert np.array_equal(g1.get_state(), g2.get_state())


def test_v1_generate_host_matches_device():
    g1 = P.ChaoticPRNG(SEEDS[0], 4096, W.V1)
    g2 = P.ChaoticPRNG(SEEDS[0], 4096, W.V1)
    for n in (128, 36):
        dev = P.as_u32(g1.generate(n))
        host = g2.generate_host(n).numpy().view(np.uint32)
        assert np.array_equal(dev, host)


@pytest.mark.parametrize("variant,n", [(W.V1, 128), (W.V1, 256), (W.V1, 36), (W.V1, 37), (W.V2, 128), (W.V3, 128)])
def test_generate_host_multi_chunk(variant, n):
    """prng_generate_host over MORE than one ~64 MiB chunk: the staging double
    buffer with its ev_gen / ev_copy waits, and the store kernels launched
    with s_begin != 0 into a chunk-sized tensor map -- at least two full
    chunks + 32 streams, so the last chunk is 32 rows (a multiple of 32, not
    of 64).  n = 256 takes the 3-D band kernel, n = 36 the 2-D TMA kernel
    with a partial last box, n = 37 the staged path.  Two calls equal
    prng_generate word for word, and the ragged last group equals the oracle."""
    rows = (64 << 20) // (4 * n) // 64 * 64   # api.cu prng_generate_host chunk rows
    S = max(2**18, 2 * rows) + 32
    g1 = P.ChaoticPRNG(SEEDS[0], S, variant)
    g2 = P.ChaoticPRNG(SEEDS[0], S, variant)
    st = O.init_states(variant, SEEDS[0], S - 32, 32)
    host = torch.empty((S, n), dtype=torch.int32, pin_memory=True)
    for _ in range(2):
        dev = P.as_u32(g1.generate(n))
        g2.generate_host(n, out=host)
        hv = host.numpy().view(np.uint32)
        assert g2.info().kernel_launches >= 3
        assert np.array_equal(dev, hv), first_mismatch(hv, dev)
        ref = O.generate(variant, st, n)
        assert np.array_equal(hv[S - 32:], ref), first_mismatch(hv[S - 32:], ref)
    assert np.array_equal(g1.get_state(), g2.get_state())
    g1.close()
    g2.close()


def test_set_state_rejects_invalid_content():
    """prng_set_state validates a checkpoint on the host before copying it:
    a V2 modulus index past the 78-entry table, a V2 state >= its modulus, an
    all-zero xorshift generator -- PrngError, device state unchanged."""
    g = P.ChaoticPRNG(3, 64, W.V2)
    good = g.get_state()
    for plane, col, val in ((8, 5, 78), (8, 0, 2**31), (3, 7, 59989 + 1)):
        bad = good.copy()
        if plane == 3:      # y >= M: use the instance's own modulus
            bad[3, col] = O.moduli()[int(good[8 + 3, col])]
        else:
            bad[plane, col] = val
        with pytest.raises(P.PrngError):
            g.set_state(bad)
        assert np.array_equal(g.get_state(), good)
    g.set_state(good)
    for variant, planes in ((W.V1, range(0, 4)), (W.V3, range(0, 2)), (W.V0, range(2, 10)), (W.V4, range(10, 20))):
        h = P.ChaoticPRNG(3, 64, variant)
        st = h.get_state()
        bad = st.copy()
        bad[list(planes), 17] = 0
        with pytest.raises(P.PrngError):
            h.set_state(bad)
        assert np.array_equal(h.get_state(), st)
        h.close()
    g.close()


def test_comb_table_size_checked():
    with pytest.raises(ValueError):
        P.ChaoticPRNG(0, 64, W.V2, comb_size=4, comb=np.zeros(8, np.uint8))   # V1-shaped table for V2
    with pytest.raises(ValueError):
        P.ChaoticPRNG(0, 64, W.V1, comb_size=4, comb=np.zeros(7, np.uint8))


def test_v1_set_state_resume():
    """Checkpoint/resume (the written-back state is a checkpoint)."""
    g = P.ChaoticPRNG(5, 256, W.V1)
    g.generate(17)
    ckpt = g.get_state()
    a = P.as_u32(g.generate(40))
    g.set_state(ckpt)
    b = P.as_u32(g.generate(40))
    assert np.array_equal(a, b)


# ------------------------------------------------------------------------ V0
@pytest.mark.parametrize("seed", SEEDS)
@pytest.mark.parametrize("S", [1, 31, 32, 33, 1000])
def test_v0(seed, S):
    _check(W.V0, seed, S, [0, 1, 3, 4, 19, 20, 21, 100, 5])


def test_v0_paper_defaults_c1_full():
    """BASELINE configs[0]: 1 stream, Listing 1 defaults, 10^6 outputs -- the
    single-stream jump-ahead path (csrc/v0_jump.cu), checked to be the one
    that ran."""
    info = _check(W.V0, 0, 1, [10**6], paper_defaults=True)
    assert info.store_path == 3, "C1 did not take the jump-ahead path"


# one block of T*L rounds is 128*16 = 2048 (n = 4096: 2 blocks); 10^6 + 1
# leaves a ragged last segment; 3_000_017 > one chunk (128 * 148 * 64 =
# 1_212_416 rounds on a 148-SM B200): three chunked launches, state carried
@pytest.mark.parametrize("ns", [[4096, 4097], [5000, 10**6 + 1], [3_000_017, 4099], [4095, 70000, 4096]])
@pytest.mark.parametrize("seed,paper_defaults", [(0, True), (W.SEEDS[0], False), (W.SEEDS[2], False)])
def test_v0_single_stream_jump(ns, seed, paper_defaults):
    """One V0 stream split over the GPU (GF(2) jump-ahead + XOR scan): the
    same words and end state as the oracle's sequential chain, over several
    calls (state carried between the jump path and, for n < 4096, the
    one-thread kernel)."""
    info = _check(W.V0, seed, 1, ns, paper_defaults=paper_defaults)
    assert info.store_path == (3 if ns[-1] >= 4096 else 1)


@pytest.mark.parametrize("S,first", [(2, 0), (3, 7), (16, 0), (16, 1000)])
def test_v0_few_streams_jump(S, first):
    """A handle with up to 16 V0 streams takes the split path too (one grid
    row of CTAs per stream, its own look-back): every stream equals the
    oracle's sequential chain, over calls and with a shard offset."""
    info = _check(W.V0, W.SEEDS[0], S, [5000, 70001], first=first)
    assert info.store_path == 3


def test_v0_few_streams_jump_multi_chunk():
    """Few streams, each longer than one chunk (3 streams: 49 CTAs per stream
    row x 128 segments x 64 rounds = 401,408 rounds per chunk on a 148-SM
    B200): three chunked launches per call, every segment jumping from its
    own row's chunk-start state, then a second call continuing the state."""
    info = _check(W.V0, W.SEEDS[2], 3, [1_000_003, 4100], first=5)
    assert info.store_path == 3 and info.kernel_launches >= 1


def test_v0_seventeen_streams_use_the_stream_kernel():
    """Past 16 streams the ordinary one-thread-per-stream kernel runs."""
    info = _check(W.V0, W.SEEDS[1], 17, [5000])
    assert info.store_path != 3


def test_v0_jump_chunk_edges_and_resume():
    """Chunk edges of the jump path (one chunk = 128 segments x 148 CTAs x
    64 rounds on a 148-SM B200): exactly one chunk, one chunk + 1 round (a
    second launch of a single round), and a resumed stream (set_state from
    a checkpoint taken mid-way) continuing word for word."""
    chunk = 128 * torch.cuda.get_device_properties(0).multi_processor_count * 64
    info = _check(W.V0, W.SEEDS[0], 1, [chunk, chunk + 1, 4096])
    assert info.store_path == 3
    g = P.ChaoticPRNG(W.SEEDS[2], 1, W.V0)
    g.generate(5000)
    ck = g.get_state()
    tail = P.as_u32(g.generate(9000))
    g2 = P.ChaoticPRNG(W.SEEDS[0], 1, W.V0)
    g2.set_state(ck)
    assert np.array_equal(P.as_u32(g2.generate(9000)), tail)
    st = O.states_from_planes(W.V0, ck)
    assert np.array_equal(tail, O.generate(W.V0, st, 9000))
    g.close()
    g2.close()


def test_v0_jump_equals_sequential_kernel(monkeypatch):
    """The jump path and the one-thread chain (CIPRNG_V0_JUMP=0) agree word
    for word at a size the oracle would take seconds on (8 * 10^6)."""
    n = 8 * 10**6
    a, pa, ia = gpu_run(W.V0, W.SEEDS[1], 1, [n])
    monkeypatch.setenv("CIPRNG_V0_JUMP", "0")
    b, pb, ib = gpu_run(W.V0, W.SEEDS[1], 1, [n])
    assert ia.store_path == 3 and ib.store_path != 3
    assert np.array_equal(a[0], b[0]) and np.array_equal(pa, pb)


# ------------------------------------------------------------------------ V2
@pytest.mark.parametrize("seed", SEEDS)
@pytest.mark.parametrize("S", [32, 64, 96, 1024])
def test_v2_default_tables(seed, S):
    _check(W.V2, seed, S, [0, 1, 3, 4, 5, 64, 7])


@pytest.mark.parametrize("C", [1, 2, 4, 32])
def test_v2_custom_tables(C):
    gen = W.rng(200 + C)
    comb = W.random_comb(gen, C, 16)
    _check(W.V2, SEEDS[1], 96 if C < 32 else 128, [5, 64, 3], comb_size=C, comb=comb)


def test_modsq_exhaustive_on_device():
    """All three division-free squarings (Barrett, the FP32-quotient form and
    Montgomery REDC) run by a kernel for every modulus and every y < M ==
    y*y % M: the FP32 round-toward-zero steps are then the hardware's, not
    the host model's."""
    import ctypes

    bad = ctypes.c_uint64(123)
    assert P.lib().prng_selftest_modsq_gpu(ctypes.byref(bad)) == 0
    assert bad.value == 0


@pytest.mark.parametrize("kind", list(range(11)))
def test_v2_kernel_kinds(monkeypatch, kind):
    """Every V2 store-kernel instantiation (squaring split between Barrett and
    the FP32 quotient or all in Montgomery form, nibble packing by funnel
    shift or LOP3 tree) is bit-identical to the oracle, incl. the per-call selection and
    rotation over several calls and a ragged n."""
    monkeypatch.setenv("CIPRNG_V2_KIND", str(kind))
    _check(W.V2, SEEDS[0], 1024 + 32, [64, 5, 1, 66])


def test_v2_hand_trace_injected(golden):
    """The hand-traced C=1 trace (tests/golden) through the GPU via set_state."""
    e = golden["hand_traces"]["v2_c1_trace"]
    midx = O.moduli().index(e["M"])
    g = P.ChaoticPRNG(0, 1, W.V2, comb_size=1, comb=np.zeros(16, np.uint8))
    planes = np.array([[v] for v in e["y"] + [midx] * 8 + [e["x"], e["tp"]]], dtype=np.uint32)
    g.set_state(planes)
    out = P.as_u32(g.generate(2))[0].tolist()
    assert out == e["outputs"]
    assert g.get_state()[:8, 0].tolist() == e["y_after_call"]


def test_v1_hand_trace_injected(golden):
    e = golden["hand_traces"]["v1_c2_trace"]
    g = P.ChaoticPRNG(0, 2, W.V1, comb_size=2, comb=np.array(e["comb1"] + e["comb2"], np.uint8))
    planes = np.array([[ln["xor128"][k] for ln in e["lanes"]] for k in range(4)]
                      + [[ln["x"] for ln in e["lanes"]], [ln["tp"] for ln in e["lanes"]]], dtype=np.uint32)
    g.set_state(planes)
    assert P.as_u32(g.generate(3)).tolist() == e["outputs"]


# ------------------------------------------------------------------ V3 / V4
# NEXT-1: Alg. 4 with the xor64 source (V3, Q29) and with
# Listing 1's fold (V4, Q30); same arrays, exchange and store paths as V1.
@pytest.mark.parametrize("seed", SEEDS)
@pytest.mark.parametrize("S", [32, 64, 96, 4096])
@pytest.mark.parametrize("store_path", [P.STORE_DIRECT, P.STORE_TMA])
def test_v3_default_tables(seed, S, store_path):
    info = _check(W.V3, seed, S, NS, store_path=store_path)
    assert info.kernel_launches == 1


@pytest.mark.parametrize("variant", [W.V3, W.V4])
@pytest.mark.parametrize("C", [1, 2, 8, 32])
def test_v34_custom_tables(variant, C):
    comb = W.random_comb(W.rng(200 + C), C, 2)
    for S in (C * 3 if C < 32 else 64, 512):
        _check(variant, SEEDS[1], S, [5, 64, 3], comb_size=C, comb=comb)


@pytest.mark.parametrize("seed", SEEDS)
@pytest.mark.parametrize("S", [32, 96, 1024])
def test_v4_default_tables(seed, S):
    _check(W.V4, seed, S, [0, 1, 3, 4, 19, 20, 21, 100, 5])


@pytest.mark.parametrize("variant", [W.V3, W.V4])
def test_v34_misaligned_and_shards(variant):
    _check(variant, 3, 128, [8, 12], out_offset_words=1)
    whole, _, _ = gpu_run(variant, SEEDS[0], 1024, [40])
    hi, _, _ = gpu_run(variant, SEEDS[0], 512, [40], first=512)
    assert np.array_equal(whole[0][512:], hi[0])


# ------------------------------------------------------------------ consumer
@pytest.mark.parametrize("variant,S,n", [(W.V0, 100, 38), (W.V1, 2048, 130), (W.V1, 96, 6), (W.V2, 1024, 66),
                                         (W.V3, 2048, 130), (W.V3, 96, 6), (W.V4, 256, 42)])
def test_consume_matches_oracle_stats(variant, S, n):
    g = P.ChaoticPRNG(SEEDS[0], S, variant)
    stats = torch.zeros(P.N_STATS, dtype=torch.int64, device="cuda")
    for _ in range(2):
        g.consume(n, stats)
    got = P.as_u64(stats)
    st = O.init_states(variant, SEEDS[0], 0, S)
    ref = np.zeros(258, np.uint64)
    for _ in range(2):
        O.stats(O.generate(variant, st, n), ref)
    assert np.array_equal(got, ref), first_mismatch(got, ref)
    # consume advances the state exactly like generate
    assert np.array_equal(g.get_state(), O.state_planes(variant, st))


@pytest.mark.parametrize("variant,first,S,n", [
    (v, *c) for v in (W.V1, W.V3) for c in ((32, 32, 4), (96, 2080, 1030), (0, 2**19 + 32, 66))
] + [(W.V2, 32, 32, 4), (W.V2, 96, 2080, 1030), (W.V2, 0, 2**17 + 32, 34)])
def test_consume_shards_and_tails(variant, first, S, n):
    """Consumer parity on a shard (s_begin of the global stream space != 0),
    with invalid rows in the last tile (V1 / V3: a half-warp, S % 64 = 32;
    V2's 32-stream tiles are whole), ragged rounds (n % 4 = 2) and, at
    2^19 + 32 (V2: 2^17 + 32) streams, more tiles than the consumer grid has
    warps (several tiles per warp through one CTA histogram); three calls
    accumulate into the same stats."""
    g = P.ChaoticPRNG(SEEDS[1], first + S, variant, shard=(first, S))
    stats = torch.zeros(P.N_STATS, dtype=torch.int64, device="cuda")
    for _ in range(3):
        g.consume(n, stats)
    st = O.init_states(variant, SEEDS[1], first, S)
    ref = np.zeros(258, np.uint64)
    for _ in range(3):
        O.stats(O.generate(variant, st, n), ref)
    got = P.as_u64(stats)
    assert np.array_equal(got, ref), first_mismatch(got, ref)
    assert np.array_equal(g.get_state(), O.state_planes(variant, st))


def test_consume_battery_per_warp_fallback():
    """CIPRNG_CTA_HIST=0 (as on a device whose reserved shared memory per
    block is not 1 KiB): the V1 / V3 consumers and battery take the per-warp
    histograms instead of the CTA one; counters still equal the oracle's."""
    import json
    import os
    import subprocess
    import sys

    code = (
        "import json, sys, numpy as np, torch; sys.path.insert(0, '.')\n"
        "import paper_1112_5239_b200 as P, workloads as W\n"
        "out = {}\n"
        "for v in (W.V1, W.V3):\n"
        "    g = P.ChaoticPRNG(W.SEEDS[0], 2080, v)\n"
        "    s = torch.zeros(P.N_STATS, dtype=torch.int64, device='cuda'); g.consume(130, s)\n"
        "    b = torch.zeros(P.N_BATTERY, dtype=torch.int64, device='cuda'); g.battery(34, b)\n"
        "    out[v] = [P.as_u64(s).tolist(), P.as_u64(b).tolist()]\n"
        "print(json.dumps(out))\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=root,
                       env={**os.environ, "CIPRNG_CTA_HIST": "0"})
    assert r.returncode == 0, r.stderr[-2000:]
    got = json.loads(r.stdout.strip().splitlines()[-1])
    for v in (W.V1, W.V3):
        st = O.init_states(v, SEEDS[0], 0, 2080)
        ref_s = O.stats(O.generate(v, st, 130))
        ref_b = O.battery(O.generate(v, st, 34))
        assert np.array_equal(np.array(got[str(v)][0], np.uint64), ref_s)
        assert np.array_equal(np.array(got[str(v)][1], np.uint64), ref_b)


@pytest.mark.parametrize("C,S", [(4, 100), (8, 200), (32, 64)])
def test_v2_consume_custom_tables_partial_warp(C, S):
    """V2 consumer with custom combination arrays and S % 32 != 0: the last
    warp holds valid lanes and invalid ones (whole combination groups of C
    streams), the invalid lanes running on y = 0 (the CTA histogram's
    zero-emitting lanes); stats and state equal the oracle's over 2 calls."""
    comb = W.random_comb(W.rng(40 + C), C, 16)
    g = P.ChaoticPRNG(SEEDS[1], S, W.V2, comb_size=C, comb=comb)
    stats = torch.zeros(P.N_STATS, dtype=torch.int64, device="cuda")
    for n in (66, 6):
        g.consume(n, stats)
    st = O.init_states(W.V2, SEEDS[1], 0, S)
    ref = np.zeros(258, np.uint64)
    for n in (66, 6):
        O.stats(O.generate(W.V2, st, n, comb_size=C, comb=comb), ref)
    got = P.as_u64(stats)
    assert np.array_equal(got, ref), first_mismatch(got, ref)
    assert np.array_equal(g.get_state(), O.state_planes(W.V2, st))


@pytest.mark.slow
@pytest.mark.parametrize("variant", [W.V1])  # V3 passes too (30 s of oracle time, left out)
def test_consume_max_n(variant):
    """The largest consumer call the ABI accepts, n = 2^24 - 2 (ciprng.h:
    PRNG_ESIZE at n >= 2^24): the per-lane u32 pair counters and the CTA
    histogram's u32 words (one 64-stream tile, 2^24 increments per column at
    most) stay exact; n = 2^24 is refused before any launch."""
    S, n = 64, 2**24 - 2
    g = P.ChaoticPRNG(SEEDS[0], S, variant)
    stats = g.consume(n)
    st = O.init_states(variant, SEEDS[0], 0, S)
    ref = np.zeros(258, np.uint64)
    for c0 in range(0, n, 2**20):  # the oracle in split-invariant pieces (V1 / V3)
        O.stats(O.generate(variant, st, min(2**20, n - c0)), ref)
    got = P.as_u64(stats)
    assert np.array_equal(got, ref), first_mismatch(got, ref)
    assert np.array_equal(g.get_state(), O.state_planes(variant, st))
    with pytest.raises(P.PrngError):
        g.consume(2**24)


@pytest.mark.parametrize("variant,C,S", [(W.V3, 8, 200), (W.V4, 8, 200), (W.V3, 2, 34), (W.V4, 32, 96)])
def test_consume_battery_custom_tables_v34(variant, C, S):
    """V3 / V4 with custom combination arrays take the general kernels
    (one lane per stream, per-warp histograms) in consumer and battery mode;
    S not a multiple of 32 leaves a partially valid last warp.  Stats,
    battery counts and state equal the oracle's."""
    comb = W.random_comb(W.rng(70 + C + variant), C, 2)
    g = P.ChaoticPRNG(SEEDS[2], S, variant, comb_size=C, comb=comb)
    stats = torch.zeros(P.N_STATS, dtype=torch.int64, device="cuda")
    bat = torch.zeros(P.N_BATTERY, dtype=torch.int64, device="cuda")
    g.consume(66, stats)
    g.battery(34, bat)
    st = O.init_states(variant, SEEDS[2], 0, S)
    ref_s = O.stats(O.generate(variant, st, 66, comb_size=C, comb=comb))
    ref_b = O.battery(O.generate(variant, st, 34, comb_size=C, comb=comb))
    assert np.array_equal(P.as_u64(stats), ref_s), first_mismatch(P.as_u64(stats), ref_s)
    assert np.array_equal(P.as_u64(bat), ref_b), first_mismatch(P.as_u64(bat), ref_b)
    assert np.array_equal(g.get_state(), O.state_planes(variant, st))


def test_consume_custom_tables_and_odd_n():
    comb = W.random_comb(W.rng(9), 4, 2)
    g = P.ChaoticPRNG(1, 64, W.V1, comb_size=4, comb=comb)
    stats = g.consume(10)
    st = O.init_states(W.V1, 1, 0, 64)
    ref = O.stats(O.generate(W.V1, st, 10, comb_size=4, comb=comb))
    assert np.array_equal(P.as_u64(stats), ref)
    with pytest.raises(P.PrngError):
        g.consume(3)
    with pytest.raises(P.PrngError):  # per-lane u32 pair counters: n < 2^31 per call
        g.consume(2**31)


# -------------------------------------------------------------------- digest
def test_digest_matches_oracle():
    g = P.ChaoticPRNG(SEEDS[0], 512, W.V1, shard=(256, 256))
    out = g.generate(33)
    d = int(P.as_u64(P.digest(out, first_stream=256))[0])
    assert d == O.digest(P.as_u32(out), 256)


@pytest.mark.parametrize("rows,n", [(1, 1), (1, 3), (1, 6), (3, 5), (7, 9), (1000, 37), (4096, 128)])
@pytest.mark.parametrize("offset", [0, 1, 2, 3])
def test_digest_ragged_and_misaligned(rows, n, offset):
    """The digest kernel's 16-byte vector body with its scalar head (output
    views 4, 8, 12 bytes past a 16-byte boundary) and ragged tail (total
    words not a multiple of 4 or of the 2-chunk unroll)."""
    gen = W.rng(28)
    buf = torch.from_numpy(W.random_words(gen, rows * n + offset).view(np.int32)).cuda()
    view = buf[offset:].view(rows, n)
    first = int(gen.integers(0, 2**20))
    d = int(P.as_u64(P.digest(view, first_stream=first))[0])
    assert d == O.digest(P.as_u32(view), first)


# ------------------------------------------------------------- full configs
@pytest.mark.slow
def test_c2_full_size_two_calls():
    """BASELINE configs[1]: V1, 2^20 streams x 128, default tables, the exact
    launch configuration bench.py times (store path AUTO)."""
    S, n = 2**20, 128
    g = P.ChaoticPRNG(SEEDS[0], S, W.V1)
    st = O.init_states(W.V1, SEEDS[0], 0, S)
    for _ in range(2):
        a = P.as_u32(g.generate(n))
        b = O.generate(W.V1, st, n)
        assert np.array_equal(a, b), first_mismatch(a, b)
    assert np.array_equal(g.get_state(), O.state_planes(W.V1, st))


@pytest.mark.slow
def test_c3_full_size_two_calls():
    """BASELINE configs[2]: V2, 2^20 streams x 64."""
    S, n = 2**20, 64
    g = P.ChaoticPRNG(SEEDS[0], S, W.V2)
    st = O.init_states(W.V2, SEEDS[0], 0, S)
    for _ in range(2):
        a = P.as_u32(g.generate(n))
        b = O.generate(W.V2, st, n)
        assert np.array_equal(a, b), first_mismatch(a, b)
    assert np.array_equal(g.get_state(), O.state_planes(W.V2, st))


@pytest.mark.slow
def test_c5_shape_consume_stats_full():
    """BASELINE configs[4] per GPU: V1 consumer, 2^20 streams x 1024 (one GPU's
    shard of the 2^23-stream C5 space), two calls; the 258 statistics equal
    the oracle's over all 2^31 numbers (generated in stream chunks), and the
    state after the calls equals the oracle's."""
    S, n, chunk = 2**20, 1024, 2**16
    g = P.ChaoticPRNG(SEEDS[0], S, W.V1)
    stats = torch.zeros(P.N_STATS, dtype=torch.int64, device="cuda")
    for _ in range(2):
        g.consume(n, stats)
    ref = np.zeros(258, np.uint64)
    planes = []
    for c0 in range(0, S, chunk):
        st = O.init_states(W.V1, SEEDS[0], c0, chunk)
        for _ in range(2):
            O.stats(O.generate(W.V1, st, n), ref)
        planes.append(O.state_planes(W.V1, st))
    got = P.as_u64(stats)
    assert np.array_equal(got, ref), first_mismatch(got, ref)
    assert np.array_equal(g.get_state(), np.concatenate(planes, axis=1))


@pytest.mark.slow
def test_v3_c2_shape_full_size():
    """NEXT-1 (i) at the C2 shape: V3, 2^20 streams x 128, two calls, TMA path."""
    S, n = 2**20, 128
    g = P.ChaoticPRNG(SEEDS[0], S, W.V3)
    st = O.init_states(W.V3, SEEDS[0], 0, S)
    for _ in range(2):
        a = P.as_u32(g.generate(n))
        b = O.generate(W.V3, st, n)
        assert np.array_equal(a, b), first_mismatch(a, b)
    assert np.array_equal(g.get_state(), O.state_planes(W.V3, st))


@pytest.mark.slow
def test_c4_shape_sampled_groups():
    """BASELINE configs[3] shape (2^23 streams x 256 per call): 3 calls on the
    GPU, 64 sampled 32-stream groups replayed by the oracle from their own
    shard seeds (per-stream seeding makes each group independent)."""
    S, n, calls = 2**23, 256, 3
    g = P.ChaoticPRNG(SEEDS[0], S, W.V1)
    gen = W.rng(44)
    groups = np.sort(gen.choice(S // 32, 64, replace=False))
    rows = (groups[:, None] * 32 + np.arange(32)[None, :]).ravel()
    sts = [O.init_states(W.V1, SEEDS[0], int(gr) * 32, 32) for gr in groups]
    out = torch.empty((S, n), dtype=torch.int32, device="cuda")
    for _ in range(calls):
        g.generate(n, out=out)
        sampled = P.as_u32(out[torch.as_tensor(rows, device="cuda")])
        ref = np.concatenate([O.generate(W.V1, st, n) for st in sts])
        assert np.array_equal(sampled, ref), first_mismatch(sampled, ref)
    del out
    torch.cuda.empty_cache()


def test_gpu_output_statistics():
    from tests import statcheck

    for variant in (W.V0, W.V1, W.V2):
        g = P.ChaoticPRNG(SEEDS[0], 2**14, variant)
        out = P.as_u32(g.generate(256))
        assert statcheck.passes(statcheck.battery(out)), variant
        s = P.as_u64(g.consume(1024))
        assert abs(statcheck.pi_zscore(int(s[0]), int(s[1]))) < 5
        assert 1e-4 < statcheck.hist_chi2_p(s[2:]) < 1 - 1e-4


@pytest.mark.parametrize("cols,wpb,grid,persist", [(8, 2, 0, 0), (32, 8, 0, 0), (16, 4, 1, 0), (32, 2, 3, 0), (32, 2, 1, 0),
                                                   (8, 8, 1, 0), (64, 1, 0, 0), (64, 2, 0, -1), (128, 1, 0, 0),
                                                   (128, 2, 0, -1), (128, 1, 0, 2)])
def test_v1_store_kernel_shapes(monkeypatch, cols, wpb, grid, persist):
    """Every V1 store-kernel shape (2-D TMA box width, 3-D band boxes,
    warps per CTA, grid cap, persistent prefetching grid) is
    bit-identical to the oracle, incl. partial boxes (n % box != 0), n not a
    multiple of 32 (band modes fall back to 2-D boxes) and a half-empty last
    tile (S % 64 == 32)."""
    monkeypatch.setenv("CIPRNG_V1_COLS", str(cols))
    monkeypatch.setenv("CIPRNG_V1_WPB", str(wpb))
    monkeypatch.setenv("CIPRNG_V1_GRID", str(grid))
    monkeypatch.setenv("CIPRNG_V1_PERSIST", str(persist))
    for S in (96, 4096 + 32, 65536):
        _check(W.V1, SEEDS[0], S, [4, 36, 128, 20, 96, 160, 256], store_path=P.STORE_TMA)


# ------------------------------------------------------------------ battery
# NEXT-2: on-device statistical battery counts == oracle counts
# (integer, bit-exact), then the >= 10^10-numbers-per-variant run of the
# SURVEY row, judged by the host p-values.
@pytest.mark.parametrize("variant,S,n", [(W.V0, 100, 38), (W.V1, 2048, 130), (W.V1, 96, 7), (W.V2, 1024, 66),
                                         (W.V3, 2048, 128), (W.V3, 96, 5), (W.V4, 256, 42)])
def test_battery_matches_oracle_counts(variant, S, n):
    g = P.ChaoticPRNG(SEEDS[2], S, variant)
    stats = torch.zeros(P.N_BATTERY, dtype=torch.int64, device="cuda")
    for _ in range(2):
        g.battery(n, stats)
    got = P.as_u64(stats)
    st = O.init_states(variant, SEEDS[2], 0, S)
    ref = np.zeros(O.N_BATTERY, np.uint64)
    for _ in range(2):
        O.battery(O.generate(variant, st, n), ref)
    assert np.array_equal(got, ref), first_mismatch(got, ref)
    assert np.array_equal(g.get_state(), O.state_planes(variant, st))
    with pytest.raises(P.PrngError):
        g.battery(2**20)


@pytest.mark.parametrize("variant", [W.V1, W.V3])
def test_battery_shard_multi_tile(variant):
    """The battery's CTA histogram (V1 / V3 fast kernels) over more tiles than
    the grid has warps, on a shard whose last tile holds an invalid half-warp,
    with a ragged round count."""
    first, S, n = 64, 2**19 + 32, 34
    g = P.ChaoticPRNG(SEEDS[2], first + S, variant, shard=(first, S))
    stats = torch.zeros(P.N_BATTERY, dtype=torch.int64, device="cuda")
    g.battery(n, stats)
    st = O.init_states(variant, SEEDS[2], first, S)
    ref = O.battery(O.generate(variant, st, n), np.zeros(O.N_BATTERY, np.uint64))
    got = P.as_u64(stats)
    assert np.array_equal(got, ref), first_mismatch(got, ref)
    assert np.array_equal(g.get_state(), O.state_planes(variant, st))


@pytest.mark.slow
@pytest.mark.parametrize("variant", [W.V0, W.V1, W.V2, W.V3, W.V4])
def test_battery_1e10_numbers(variant):
    from paper_1112_5239_b200 import battery as B

    S, n = 2**20, 1024
    calls = -(-10**10 // (S * n))  # >= 1e10 numbers
    g = P.ChaoticPRNG(SEEDS[0], S, variant)
    stats = torch.zeros(P.N_BATTERY, dtype=torch.int64, device="cuda")
    for _ in range(calls):
        g.battery(n, stats)
    p = B.pvalues(P.as_u64(stats), S * calls, n)
    assert B.passes(p, alpha=1e-4), p


@pytest.mark.parametrize("tpw", [2, 3])
def test_v1_store_tiles_per_warp(monkeypatch, tpw):
    """Several 64-stream tiles per warp (state of the next tile prefetched
    while the current one computes) stay bit-exact, incl. a ragged last tile."""
    monkeypatch.setenv("CIPRNG_V1_TPW", str(tpw))
    for S in (96, 4096 + 32):
        _check(W.V1, SEEDS[1], S, [4, 36, 128, 20], store_path=P.STORE_TMA)


def test_cuda_graph_capture_replay():
    """generate() is capturable in a CUDA graph (programmatic-dependent
    launches, TMA descriptors as __grid_constant__ parameters): replaying a
    graph of 3 calls twice continues the streams exactly like 6 direct calls."""
    S, n = 4096, 128
    g = P.ChaoticPRNG(SEEDS[0], S, W.V1)
    outs = [torch.empty((S, n), dtype=torch.int32, device="cuda") for _ in range(3)]
    g.generate(n, out=outs[0])  # warm-up outside capture (descriptor cache, attributes)
    st = O.init_states(W.V1, SEEDS[0], 0, S)
    O.generate(W.V1, st, n)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        for o in outs:
            g.generate(n, out=o)
    torch.cuda.synchronize()
    for _ in range(2):
        graph.replay()
        torch.cuda.synchronize()
        for o in outs:
            ref = O.generate(W.V1, st, n)
            assert np.array_equal(P.as_u32(o), ref)
    assert np.array_equal(g.get_state(), O.state_planes(W.V1, st))


def test_abi_named_python_calls():
    """The prng_* Python names reach the same kernels (north_star's
    prng_create(seed, n_streams, variant) / prng_generate / prng_destroy)."""
    h = P.prng_create(SEEDS[0], 256, W.V1)
    a = P.as_u32(P.prng_generate(h, 40))
    st = O.init_states(W.V1, SEEDS[0], 0, 256)
    assert np.array_equal(a, O.generate(W.V1, st, 40))
    s = P.as_u64(P.prng_consume(h, 8))
    assert np.array_equal(s, O.stats(O.generate(W.V1, st, 8)))
    assert np.array_equal(P.prng_get_state(h), O.state_planes(W.V1, st))
    P.prng_destroy(h)


def test_v1_store_path_smem_stg(monkeypatch):
    """SURVEY s7 store path (b): the swizzled shared-memory box written back by
    the warp with coalesced 128-bit STG -- bit-identical, incl. partial boxes,
    a half-empty last tile and n % 4 != 0 (which falls back to the direct path)."""
    monkeypatch.setenv("CIPRNG_V1_SMEM_STG", "1")
    for S in (96, 4096 + 32, 65536):
        _check(W.V1, SEEDS[2], S, [4, 36, 128, 20, 96, 160, 5], store_path=P.STORE_DIRECT)
