"""Pins of the CPU oracle to things other than itself (not gpu).

Each test names what fixes the value: the paper's worked example, a published
sequence of a generator the paper cites, a hand trace under tests/golden/, an
invariant the paper states, a special case, or brute force.  Readings Qn are
listed in DESIGN.md s3.
"""
import math

import numpy as np
import pytest

import oracle as O
import workloads as W
from tests import statcheck

M32 = 0xFFFFFFFF


# ---------------------------------------------------------------- Eq. Oplus
def test_table1_round(golden):
    """Table 1: the paper's worked x XOR S^i."""
    g = golden["table1"]
    x, s, r = (int(g[k], 2) for k in ("x", "S", "x_xor_S"))
    assert O.xor_step(x, s) == r


def test_oplus_special_cases():
    """x ^ 0 = x; (x ^ s) ^ s = x; exactly the bits set in S flip."""
    gen = W.rng(1)
    for x, s in W.random_words(gen, (64, 2)).tolist():
        assert O.xor_step(x, 0) == x
        assert O.xor_step(O.xor_step(x, s), s) == x
        assert bin(O.xor_step(x, s) ^ x).count("1") == bin(s).count("1")


# ------------------------------------------------------- strategy sources
def test_xorshift32_alg2(golden):
    p = golden["published_sequences"]
    for key in ("xorshift32_13_17_5", "xorshift32_from_1"):
        e = p[key]
        assert O.xorshift32_seq(e["seed"], len(e["outputs"])) == e["outputs"]


def test_xor64_published(golden):
    e = golden["published_sequences"]["xor64"]
    assert O.xor64_seq(e["seed"], len(e["outputs"])) == e["outputs"]


def test_xor128_32_published(golden):
    e = golden["published_sequences"]["xor128_32"]
    assert O.xor128_32_seq(e["seed"], len(e["outputs"])) == e["outputs"]


def test_xor128_64_and_xorwow_64_hand(golden):
    h = golden["hand_traces"]
    e = h["xor128_64_tiny"]
    assert O.xor128_64_seq(e["state"], 2) == e["outputs"]
    e = h["xorwow_64_tiny"]
    assert O.xorwow_64_seq(e["state"], e["d"], 2) == e["outputs"]


# ----------------------------------------------------------------- seeder
def test_splitmix_published(golden):
    e = golden["published_sequences"]["splitmix64"]
    assert [O.splitmix_word(e["seed"], 0, k) for k in range(5)] == e["outputs"]


def test_splitmix_counter_structure():
    """W(seed, s, k) is output 16*s+k+1 of one SplitMix64 sequence: the word
    for (s, k) equals the word for (0, 16*s + k) (Q11; stream-count invariance
    rests on this)."""
    for s in (1, 7, 12345):
        for k in (0, 5, 15):
            assert O.splitmix_word(99, s, k) == O.splitmix_word(99, 0, 16 * s + k)
    assert O.mix64(0) == 0  # fixed point of the finaliser


# --------------------------------------------------------------------- V0
def _v0_state(a, b, c, d, x):
    st = np.zeros((1, 24), dtype=np.uint32)
    for i, v in enumerate([a, *b, *c, d]):
        st[0, 2 * i] = v & M32
        st[0, 2 * i + 1] = v >> 32
    st[0, 22] = x
    return st


def test_v0_hand_trace(golden):
    e = golden["hand_traces"]["v0_tiny_first_output"]
    s = e["state"]
    st = _v0_state(s["a"], s["b"], s["c"], s["d"], s["x"])
    assert O.generate(O.V0, st, 1)[0].tolist() == e["outputs"]


def test_v0_paper_defaults_is_listing1_fold():
    """I1 for V0: x_i ^ x_{i-1} = lo^hi fold of the three pinned generators
    (Listing 1), starting from x = 123123123."""
    n = 64
    st = O.init_states(O.V0, 0, 0, 1, paper_defaults=True)
    out = O.generate(O.V0, st, n)[0].astype(np.uint64)
    t1 = O.xor64_seq(88172645463325252, n)
    t2 = O.xor128_64_seq([123456789, 362436069, 521288629, 88675123], n)
    t3 = O.xorwow_64_seq([123456789, 362436069, 521288629, 88675123, 5783321], 6615241, n)
    prev = 123123123
    for i in range(n):
        f = 0
        for t in (t1[i], t2[i], t3[i]):
            f ^= (t & M32) ^ (t >> 32)
        assert int(out[i]) == prev ^ f
        prev = int(out[i])


def test_v0_split_invariance():
    """I4: generate(a+b) == generate(a) ++ generate(b) (state persists)."""
    st1 = O.init_states(O.V0, 5, 0, 3)
    st2 = st1.copy()
    full = O.generate(O.V0, st1, 10)
    part = np.concatenate([O.generate(O.V0, st2, 4), O.generate(O.V0, st2, 6)], axis=1)
    assert np.array_equal(full, part)
    assert np.array_equal(st1, st2)


def test_v0_paper_defaults_needs_single_stream():
    with pytest.raises(O.OracleError):
        O.init_states(O.V0, 0, 0, 2, paper_defaults=True)


# --------------------------------------------------------------------- V1
def test_v1_hand_trace_c2(golden):
    e = golden["hand_traces"]["v1_c2_trace"]
    st = np.array([[*ln["xor128"], ln["x"], ln["tp"]] for ln in e["lanes"]], dtype=np.uint32)
    comb = np.array(e["comb1"] + e["comb2"], dtype=np.uint8)
    out = O.generate(O.V1, st, 3, comb_size=2, comb=comb)
    assert out.tolist() == e["outputs"]


def test_v1_self_combination_is_prefix_xor_of_xor128(golden):
    """I2 + I1: with C = 1 (o1 = o2 = self) the shared terms cancel,
    so x_i = x_{i-1} ^ xor128(), the published Marsaglia sequence."""
    seeds = golden["published_sequences"]["xor128_32"]["seed"]
    x0 = 0xDEADBEEF
    st = np.array([[*seeds, x0, 0x12345678]], dtype=np.uint32)
    out = O.generate(O.V1, st, 5, comb_size=1, comb=np.array([0, 0], dtype=np.uint8))[0]
    assert int(out[0]) == x0 ^ golden["published_sequences"]["xor128_32"]["outputs"][0]
    g = O.xor128_32_seq(seeds, 5)
    prev = x0
    for i in range(5):
        assert int(out[i]) == prev ^ g[i]
        prev = int(out[i])


def _xor128_streams(st, n):
    return np.array([O.xor128_32_seq(row[:4].tolist(), n) for row in st], dtype=np.uint64)


@pytest.mark.parametrize("custom", [False, True])
def test_v1_group_parity(custom):
    """I3: comb1, comb2 are permutations, so every previous-round t is used
    exactly twice per group and XOR over lanes of t_i equals XOR over lanes of
    the xor-like draws g_i; with I1 (x_i ^ x_{i-1} = t_i) this is checkable
    from the outputs and the pinned xor128 alone."""
    gen = W.rng(3)
    S, n = 64, 9
    st = O.init_states(O.V1, 77, 0, S)
    x0 = st[:, 4].astype(np.uint64)
    comb = W.random_comb(gen, 32, 2) if custom else None
    g = _xor128_streams(st, n)
    out = O.generate(O.V1, st.copy(), n, comb=comb).astype(np.uint64)
    t = out ^ np.concatenate([x0[:, None], out[:, :-1]], axis=1)
    for grp in range(S // 32):
        sl = slice(32 * grp, 32 * grp + 32)
        assert np.array_equal(np.bitwise_xor.reduce(t[sl], axis=0), np.bitwise_xor.reduce(g[sl], axis=0))


def test_v1_default_tables_plus1_plus17():
    """Reading Q6: the default arrays are comb1[l] = l+1, comb2[l] = l+17 (mod
    32).  Inject a single non-zero shared cell at lane k: in round 0 exactly
    lanes k-1 and k-17 see it (t = g ^ shmem[o1] ^ shmem[o2])."""
    S = 32
    st = O.init_states(O.V1, 1, 0, S)
    st[:, 4] = 0
    st[:, 5] = 0
    k, T = 20, 0xA5A5A5A5
    st[k, 5] = T
    g = _xor128_streams(st, 1)[:, 0]
    out = O.generate(O.V1, st, 1)[:, 0].astype(np.uint64)
    seen = {l for l in range(S) if int(out[l] ^ g[l]) == T}
    zero = {l for l in range(S) if int(out[l] ^ g[l]) == 0}
    assert seen == {(k - 1) % 32, (k - 17) % 32}
    assert zero == set(range(S)) - seen


def test_v1_split_invariance():
    st1 = O.init_states(O.V1, 9, 0, 64)
    st2 = st1.copy()
    full = O.generate(O.V1, st1, 13)
    part = np.concatenate([O.generate(O.V1, st2, 5), O.generate(O.V1, st2, 8)], axis=1)
    assert np.array_equal(full, part) and np.array_equal(st1, st2)


def test_v1_shard_invariance():
    """I5: per-stream seeding makes a shard's output its slice of the whole."""
    whole = O.generate(O.V1, O.init_states(O.V1, 4, 0, 128), 7)
    hi = O.generate(O.V1, O.init_states(O.V1, 4, 64, 64), 7)
    assert np.array_equal(whole[64:], hi)


def test_v1_config_errors():
    st = O.init_states(O.V1, 0, 0, 33)
    with pytest.raises(O.OracleError):
        O.generate(O.V1, st, 1)  # incomplete group
    st = O.init_states(O.V1, 0, 0, 4)
    with pytest.raises(O.OracleError):
        O.generate(O.V1, st, 1, comb_size=4, comb=np.array([0, 1, 2, 4, 0, 1, 2, 3], np.uint8))
    with pytest.raises(O.OracleError):
        O.generate(O.V1, st, 1, comb_size=4)  # defaults exist for C = 32 only


# --------------------------------------------------------------------- V2
def _v2_state(y, midx, x, tp):
    return np.array([[*y, *midx, x, tp]], dtype=np.uint32)


def test_bbs_small(golden):
    for c in golden["hand_traces"]["bbs_small"]["cases"]:
        y, orbit = c["y"], []
        for _ in c["orbit"]:
            y = O.bbs_step(y, c["M"])
            orbit.append(y)
        assert orbit == c["orbit"]


def test_modulus_table_constraints():
    """Q13 / P:1212-1214: products of two distinct primes = 3 (mod 4) 'around
    256', M < 2^16, so x^2 < 2^32 with 32-bit arithmetic."""
    mods = O.moduli()
    primes = [p for p in range(128, 257) if all(p % d for d in range(2, int(p**0.5) + 1)) and p % 4 == 3]
    assert len(primes) == 13 and len(mods) == 78 == math.comb(13, 2)
    assert mods == sorted(mods) and mods[0] == 131 * 139 and mods[-1] == 239 * 251 == 59989
    for M in mods:
        assert M < 2**16 and (M - 1) ** 2 < 2**32
        fac = [p for p in primes if M % p == 0]
        assert len(fac) == 2 and fac[0] * fac[1] == M


def test_v2_hand_trace_c1(golden):
    e = golden["hand_traces"]["v2_c1_trace"]
    midx = O.moduli().index(e["M"])
    st = _v2_state(e["y"], [midx] * 8, e["x"], e["tp"])
    out = O.generate(O.V2, st, 2, comb_size=1, comb=np.zeros(16, np.uint8))
    assert out[0].tolist() == e["outputs"]
    assert st[0, :8].tolist() == e["y_after_call"]


def test_v2_rotation_direction():
    """'internal variable for BBS number 1 is stored in place 2,
    ..., BBS number 8 is stored in place 1' -- and the modulus moves with it
    (Q19).  Per round instances 1, 2, 3, 7 are drawn twice, the others once
    (P:1269-1280)."""
    mods = O.moduli()
    st = O.init_states(O.V2, 11, 0, 32)
    before = st.copy()
    O.generate(O.V2, st, 1)
    draws = [2, 2, 2, 1, 1, 1, 2, 1]
    for s in range(32):
        for j in range(8):
            y, m = int(before[s, j]), int(before[s, 8 + j])
            for _ in range(draws[j]):
                y = y * y % mods[m]
            assert int(st[s, (j + 1) % 8]) == y and int(st[s, 8 + (j + 1) % 8]) == m


def test_v2_zero_rounds_no_rotation():
    st = O.init_states(O.V2, 2, 0, 32)
    before = st.copy()
    out = O.generate(O.V2, st, 0)
    assert out.shape == (32, 0) and np.array_equal(st, before)


def test_v2_state_invariants():
    """I6: 1 < y < M-1, gcd(y, M) = 1, y^2 < 2^32, across calls."""
    mods = O.moduli()
    st = O.init_states(O.V2, 3, 0, 64)
    for _ in range(20):
        for row in st:
            for j in range(8):
                y, M = int(row[j]), mods[int(row[8 + j])]
                assert 1 < y < M - 1 and math.gcd(y, M) == 1 and y * y < 2**32
        O.generate(O.V2, st, 37)


def test_v2_selection_uses_call_entry_states():
    """Q15/Q16: o1 = comb[bbs1 & 7], o2 = comb[8 + (bbs2 & 7)]
    with the call-entry states; default arrays are l+1+a and l+17+a (Q6).
    Inject one non-zero shared cell at lane k and predict who sees it."""
    st = O.init_states(O.V2, 21, 0, 32)
    st[:, 16] = 0
    st[:, 17] = 0
    k, T = 5, 0x5A5A5A5A
    st[k, 17] = T
    entry = st.copy()
    # each lane's own strategy word from a self-cancelling C=1 run (pinned above)
    own = np.zeros(32, dtype=np.uint64)
    for l in range(32):
        one = entry[l : l + 1].copy()
        one[0, 17] = 0
        own[l] = O.generate(O.V2, one, 1, comb_size=1, comb=np.zeros(16, np.uint8))[0, 0]
    out = O.generate(O.V2, st, 1)[:, 0].astype(np.uint64)
    for l in range(32):
        o1 = (l + 1 + (int(entry[l, 0]) & 7)) % 32
        o2 = (l + 17 + (int(entry[l, 1]) & 7)) % 32
        expect = (T if o1 == k else 0) ^ (T if o2 == k else 0)
        assert int(out[l] ^ own[l]) == expect


def test_v2_not_split_invariant():
    """I4 negative: selection and rotation happen per call (P:1224-1230,
    P:1287), so two calls of 3 differ from one call of 6."""
    st1 = O.init_states(O.V2, 8, 0, 32)
    st2 = st1.copy()
    full = O.generate(O.V2, st1, 6)
    part = np.concatenate([O.generate(O.V2, st2, 3), O.generate(O.V2, st2, 3)], axis=1)
    assert np.array_equal(full[:, :3], part[:, :3])
    assert not np.array_equal(full, part)


# ------------------------------------------------------------ consumer stats
def test_stats_brute_force():
    gen = W.rng(5)
    words = W.random_words(gen, (7, 10))
    words[0, 0], words[0, 1] = 0xFFFFFFFF, 0  # boundary pair: u^2 < 2^64
    words[1, 0], words[1, 1] = 0xFFFFFFFF, 1  # u^2 + v^2 > 2^64 - 1? check exactly
    st = O.stats(words)
    inside = pairs = 0
    hist = [0] * 256
    for row in words.tolist():
        for v in row:
            hist[v >> 24] += 1
        for i in range(0, len(row), 2):
            pairs += 1
            inside += row[i] ** 2 + row[i + 1] ** 2 < 2**64
    assert int(st[0]) == inside and int(st[1]) == pairs and st[2:].tolist() == hist


def test_stats_odd_n_rejected():
    with pytest.raises(O.OracleError):
        O.stats(np.zeros((2, 3), np.uint32))


@pytest.mark.parametrize("variant", [O.V0, O.V1, O.V2, O.V3, O.V4])
def test_oracle_output_statistics(variant):
    """Frequency / runs / byte chi-square sanity (stand-in for BigCrush,
    P:851-853) and the Monte-Carlo pi estimate within 5 sigma."""
    S, n = (32, 4096) if variant else (8, 16384)
    st = O.init_states(variant, W.SEEDS[0], 0, S)
    out = O.generate(variant, st, n)
    assert statcheck.passes(statcheck.battery(out))
    s = O.stats(out)
    assert abs(statcheck.pi_zscore(int(s[0]), int(s[1]))) < 5
    assert 1e-4 < statcheck.hist_chi2_p(s[2:]) < 1 - 1e-4


def test_statcheck_negative_controls():
    """all-zero and alternating streams must fail."""
    assert not statcheck.passes(statcheck.battery(np.zeros(4096, np.uint32)))
    assert not statcheck.passes(statcheck.battery(np.full(4096, 0x55555555, np.uint32)))


def test_digest_shard_additive():
    """Q28: the digest is a position-aware sum, so shard digests add mod 2^64."""
    out = O.generate(O.V1, O.init_states(O.V1, 1, 0, 64), 8)
    assert O.digest(out) == (O.digest(out[:32]) + O.digest(out[32:], 32)) % 2**64
    swapped = out.copy()
    swapped[[0, 1]] = swapped[[1, 0]]
    assert O.digest(swapped) != O.digest(out)
    swapped = out.copy()
    swapped[5, [2, 3]] = swapped[5, [3, 2]]
    assert swapped[5, 2] != swapped[5, 3] and O.digest(swapped) != O.digest(out)


def test_digest_pairs_are_published_splitmix64(golden):
    """Q28: h = output number P of SplitMix64 seeded with the word pair (hi:lo),
    P the pair's global position, so a one-pair row (seed, 0) -- or a lone
    word of an odd row, paired with 0 -- at pair position k + 1 digests to the
    k-th published SplitMix64 output for that seed (tests/golden: 1234567)."""
    e = golden["published_sequences"]["splitmix64"]
    assert e["seed"] < 2**32  # the seed fits the low word
    for k, want in enumerate(e["outputs"]):
        assert O.digest(np.array([[e["seed"], 0]], np.uint32), k + 1) == want  # n = 2: P = first_stream
        assert O.digest(np.array([[e["seed"]]], np.uint32), k + 1) == want     # n = 1: lone word, hi = 0
    # rows are whole units: rows 1..5 of a one-word-per-row block sum the sequence
    rows = np.full((5, 1), e["seed"], np.uint32)
    assert O.digest(rows, 1) == sum(e["outputs"]) % 2**64


def test_digest_injective_in_word():
    """Q28: for a fixed position h(idx, .) is a bijection of the word (add,
    xorshift and odd multiply are invertible), so one wrong word always
    changes the digest: 2^16 distinct words at one position, at two
    positions, give 2^16 distinct digests."""
    for first, n in ((0, 1), (12345, 7)):
        words = np.arange(0, 2**32, 2**16, dtype=np.uint64).astype(np.uint32)
        ds = {O.digest(np.array([[w]], np.uint32), first * n) for w in words} if n == 1 else \
            {O.digest(np.full((1, n), w, np.uint32), first) for w in words[:4096]}
        assert len(ds) == (len(words) if n == 1 else 4096)


# ---------------------------------------------------------------- V3 / V4
# NEXT-1: Alg. 4's combination with the xor64 of the paper's
# "optimized versions" (V3, reading Q29) and with Listing 1's
# three-generator fold (V4, reading Q30).
def _v3_state(rows):
    """rows of (a, x, tp) -> oracle structs (a.lo, a.hi, x, tp)."""
    return np.array([[a & M32, a >> 32, x, tp] for a, x, tp in rows], dtype=np.uint32)


def test_v3_hand_trace_c2(golden):
    e = golden["hand_traces"]["v3_c2_trace"]
    st = _v3_state([(ln["a"], ln["x"], ln["tp"]) for ln in e["lanes"]])
    comb = np.array(e["comb1"] + e["comb2"], dtype=np.uint8)
    out = O.generate(O.V3, st, 2, comb_size=2, comb=comb)
    assert out.tolist() == e["outputs"]
    assert [int(r[0]) | int(r[1]) << 32 for r in st] == e["a_after"]


def test_v3_self_combination_is_prefix_xor_of_xor64(golden):
    """I2 + I1 with C = 1: x_i = x_{i-1} ^ lo32(xor64_i); the first draw is the
    published Marsaglia value from its published seed."""
    e = golden["published_sequences"]["xor64"]
    x0 = 0x0BADF00D
    st = _v3_state([(e["seed"], x0, 0x77777777)])
    out = O.generate(O.V3, st, 6, comb_size=1, comb=np.array([0, 0], np.uint8))[0]
    assert int(out[0]) == x0 ^ (e["outputs"][0] & M32)
    prev = x0
    for i, a in enumerate(O.xor64_seq(e["seed"], 6)):
        assert int(out[i]) == prev ^ (a & M32)
        prev = int(out[i])


@pytest.mark.parametrize("variant", [O.V3, O.V4])
@pytest.mark.parametrize("custom", [False, True])
def test_v34_group_parity(variant, custom):
    """I3 as for V1: XOR over a group's lanes of t_i equals XOR of the draws
    g_i, which a C = 1 run (I2: t = g) of the same states exposes."""
    S, n = 64, 7
    st = O.init_states(variant, 31, 0, S)
    xcol = 2 if variant == O.V3 else 22
    x0 = st[:, xcol].astype(np.uint64)
    solo = st.copy()
    g = O.generate(variant, solo, n, comb_size=1, comb=np.zeros(2, np.uint8)).astype(np.uint64)
    g ^= np.concatenate([x0[:, None], g[:, :-1]], axis=1)
    comb = W.random_comb(W.rng(4), 32, 2) if custom else None
    out = O.generate(variant, st, n, comb=comb).astype(np.uint64)
    t = out ^ np.concatenate([x0[:, None], out[:, :-1]], axis=1)
    for grp in range(S // 32):
        sl = slice(32 * grp, 32 * grp + 32)
        assert np.array_equal(np.bitwise_xor.reduce(t[sl], axis=0), np.bitwise_xor.reduce(g[sl], axis=0))


def test_v4_self_combination_is_listing1():
    """I2 for V4: with C = 1 the shared terms cancel, so V4 is exactly Listing 1
    (= V0, pinned above to its hand trace and to the fold of the published
    generators) when both start from the same generator words and x."""
    v0 = O.init_states(O.V0, 0, 0, 1, paper_defaults=True)
    v4 = np.zeros((1, 24), np.uint32)
    v4[0, :23] = v0[0, :23]
    v4[0, 23] = 0xCAFEBABE  # tp: cancels
    a = O.generate(O.V0, v0, 40)
    b = O.generate(O.V4, v4, 40, comb_size=1, comb=np.zeros(2, np.uint8))
    assert np.array_equal(a, b)
    assert np.array_equal(v0[0, :23], v4[0, :23])


@pytest.mark.parametrize("variant", [O.V3, O.V4])
def test_v34_default_tables_plus1_plus17(variant):
    """Q6 defaults shared with V1: a single injected shared cell at lane k
    reaches exactly lanes k-1 and k-17 in round 0."""
    S = 32
    st = O.init_states(variant, 3, 0, S)
    xcol = 2 if variant == O.V3 else 22
    st[:, xcol] = 0
    st[:, xcol + 1] = 0
    solo = st.copy()
    g = O.generate(variant, solo, 1, comb_size=1, comb=np.zeros(2, np.uint8))[:, 0].astype(np.uint64)
    k, T = 9, 0x3C3C3C3C
    st[k, xcol + 1] = T
    out = O.generate(variant, st, 1)[:, 0].astype(np.uint64)
    assert {l for l in range(S) if int(out[l] ^ g[l]) == T} == {(k - 1) % 32, (k - 17) % 32}
    assert {l for l in range(S) if int(out[l] ^ g[l]) == 0} == set(range(S)) - {(k - 1) % 32, (k - 17) % 32}


@pytest.mark.parametrize("variant", [O.V3, O.V4])
def test_v34_split_and_shard_invariance(variant):
    st1 = O.init_states(variant, 9, 0, 64)
    st2 = st1.copy()
    full = O.generate(variant, st1, 11)
    part = np.concatenate([O.generate(variant, st2, 4), O.generate(variant, st2, 7)], axis=1)
    assert np.array_equal(full, part) and np.array_equal(st1, st2)
    hi = O.generate(variant, O.init_states(variant, 9, 32, 32), 11)
    assert np.array_equal(full[32:], hi)


def test_v34_seeding():
    """Seeds (Q11 extended): V3 a = W(s,0), x = lo W(s,1), tp = lo W(s,2); V4
    shares V0's generator words and takes x = lo W(s,11), tp = lo W(s,12)."""
    st = O.init_states(O.V3, 5, 7, 2)
    for r, s in enumerate((7, 8)):
        a = O.splitmix_word(5, s, 0)
        assert [int(v) for v in st[r]] == [a & M32, a >> 32, O.splitmix_word(5, s, 1) & M32,
                                          O.splitmix_word(5, s, 2) & M32]
    v4 = O.init_states(O.V4, 5, 7, 2)
    v0 = O.init_states(O.V0, 5, 7, 2)
    assert np.array_equal(v4[:, :22], v0[:, :22])
    assert v4[:, 22].tolist() == [O.splitmix_word(5, s, 11) & M32 for s in (7, 8)]
    assert v4[:, 23].tolist() == [O.splitmix_word(5, s, 12) & M32 for s in (7, 8)]


def test_survey_vectors(golden):
    """SURVEY.md Appendix A's independently computed vectors (see the golden
    file's note): generator prefixes and Listing 1's first outputs."""
    g = golden["survey_vectors"]
    assert O.xor64_seq(g["xor64_first3"]["seed"], 3) == g["xor64_first3"]["outputs"]
    assert O.xor128_32_seq(g["xor128_32_first5"]["seed"], 5) == g["xor128_32_first5"]["outputs"]
    assert O.xor128_64_seq(g["xor128_64_first2"]["seed"], 2) == g["xor128_64_first2"]["outputs"]
    e = g["xorwow_64_first2"]
    assert O.xorwow_64_seq(e["seed"], e["d"], 2) == e["outputs"] == e["published_32bit_xorwow"][:2]
    st = O.init_states(O.V0, 0, 0, 1, paper_defaults=True)
    assert O.generate(O.V0, st, 4)[0].tolist() == g["listing1_paper_defaults_first4"]["outputs"]


# ------------------------------------------------ seeders (Q11, Q12, Q21)
# The word -> state mapping of every variant, pinned to the published
# SplitMix64 sequence (test_splitmix_published) through O.splitmix_word, and
# its zero guards / rejection loop reached by injecting words
# (O.init_from_words, the oracle's test hook).  Marsaglia's seeds are the
# literals of the published code (tests/golden/published_sequences.json).
MARS128 = [123456789, 362436069, 521288629, 88675123]
XOR64_SEED = 88172645463325252


def _u64(lo, hi):
    return int(lo) | (int(hi) << 32)


def _v0_fields(row):
    """orc_v0_state as u32 words: a, b[4], c[5], d (u64 lo/hi pairs), x, pad."""
    r = [int(v) for v in row]
    u = [_u64(r[2 * k], r[2 * k + 1]) for k in range(11)]
    return {"a": u[0], "b": u[1:5], "c": u[5:10], "d": u[10], "x": r[22]}


@pytest.mark.parametrize("seed", W.SEEDS)
def test_v0_seeding_word_mapping(seed):
    """Q11/Q12: a = W(s,0), b = W(s,1..4), c = W(s,5..9), d = W(s,10),
    x = lo W(s,11) -- W read from the published SplitMix64 generator."""
    st = O.init_states(O.V0, seed, 1000, 3)
    for r, s in enumerate(range(1000, 1003)):
        w = [O.splitmix_word(seed, s, k) for k in range(12)]
        f = _v0_fields(st[r])
        assert f["a"] == w[0] and f["b"] == w[1:5] and f["c"] == w[5:10] and f["d"] == w[10]
        assert f["x"] == w[11] & M32 and int(st[r, 23]) == 0


def test_splitmix_word_is_published_generator_output():
    """W(seed, s, k) is output number 16s+k+1 of SplitMix64 run from `seed`:
    iterate the published recurrence (state += golden gamma, then mix) in
    Python big integers and read outputs 17..32 as stream 1's words."""
    seed, state, outs = 0xDEADBEEF, 0xDEADBEEF, []
    for _ in range(48):
        state = (state + 0x9E3779B97F4A7C15) % 2**64
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) % 2**64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) % 2**64
        outs.append(z ^ (z >> 31))
    for s in range(3):
        assert [O.splitmix_word(seed, s, k) for k in range(16)] == outs[16 * s:16 * s + 16]


def test_v0_zero_guards_injected():
    """An all-zero xorshift state is a fixed point (every step maps 0 to 0),
    so each generator whose seeder words are all zero restarts from
    Marsaglia's published seeds; the guarded states then reproduce the
    published first outputs.  Guards are per generator and only fire on an
    all-zero state."""
    f = _v0_fields(O.init_from_words(O.V0, [0] * 16))
    assert f["a"] == XOR64_SEED and f["b"] == MARS128 and f["c"] == MARS128 + [5783321]
    assert f["d"] == 0 and f["x"] == 0
    assert O.xor64_seq(f["a"], 1) == [8748534153485358512]
    # only the xor128 block zero: the others keep their words
    w = [7] + [0, 0, 0, 0] + [1, 2, 3, 4, 5, 99, 0xABCDEF0123456789]
    f = _v0_fields(O.init_from_words(O.V0, w))
    assert f["a"] == 7 and f["b"] == MARS128 and f["c"] == [1, 2, 3, 4, 5] and f["d"] == 99
    assert f["x"] == 0x23456789
    # a single non-zero word (even only in the high half) is not guarded
    w = [0, 0, 0, 0, 1 << 40, 0, 0, 0, 0, 1 << 63, 0, 0]
    f = _v0_fields(O.init_from_words(O.V0, w))
    assert f["a"] == XOR64_SEED and f["b"] == [0, 0, 0, 1 << 40] and f["c"] == [0, 0, 0, 0, 1 << 63]


@pytest.mark.parametrize("seed", W.SEEDS)
def test_v1_seeding_word_mapping(seed):
    """Q8/Q11: xor128 (a,b,c,d) = lo W(s,0..3), x = lo W(s,4), tp = lo W(s,5)."""
    st = O.init_states(O.V1, seed, 77, 3)
    for r, s in enumerate(range(77, 80)):
        assert [int(v) for v in st[r]] == [O.splitmix_word(seed, s, k) & M32 for k in range(6)]


def test_v1_zero_guard_on_low_words():
    """The xor128-32 state is the LOW halves of W(s,0..3): words whose low
    halves are all zero (high halves not) give the all-zero 32-bit state and
    must take Marsaglia's seeds -> first output 3701687786 (published)."""
    st = O.init_from_words(O.V1, [1 << 32, 5 << 40, 0, 1 << 63, 0x1_0000_0011, 0x2_0000_0022])
    assert [int(v) for v in st] == MARS128 + [0x11, 0x22]
    assert O.xor128_32_seq(MARS128, 1) == [3701687786]
    st = O.init_from_words(O.V1, [0, 0, 0, 9, 1, 2])
    assert [int(v) for v in st] == [0, 0, 0, 9, 1, 2]


def test_v3_v4_zero_guards_injected():
    st = O.init_from_words(O.V3, [0, 0xAAAA_BBBB_CCCC_DDDD, 3])
    assert _u64(st[0], st[1]) == XOR64_SEED and int(st[2]) == 0xCCCCDDDD and int(st[3]) == 3
    v4 = O.init_from_words(O.V4, [0] * 11 + [5, 6])
    v0 = O.init_from_words(O.V0, [0] * 11 + [5, 6])
    assert np.array_equal(v4[:22], v0[:22]) and int(v4[22]) == 5 and int(v4[23]) == 6


def _bbs_moduli_independent():
    """Q13 re-derived here: products p < q of the primes = 3 (mod 4) in
    [128, 256], ascending."""
    primes = [p for p in range(128, 257) if p % 4 == 3 and all(p % d for d in range(2, p))]
    return sorted(p * q for i, p in enumerate(primes) for q in primes[i + 1:]), primes


def _q21_seed(w, mods):
    """Q21 written out: modulus index hi(w) mod 78, r = 2 + lo(w) mod (M-3),
    stepped until gcd(r, M) = 1 and r^2 mod M > 1; state y = r^2 mod M."""
    mi = (w >> 32) % len(mods)
    M = mods[mi]
    r = 2 + (w & M32) % (M - 3)
    while math.gcd(r, M) != 1 or pow(r, 2, M) <= 1:
        r = 2 if r == M - 2 else r + 1
    return pow(r, 2, M), mi, r


@pytest.mark.parametrize("seed", W.SEEDS)
def test_v2_seeding_q21_and_quadratic_residues(seed):
    """BBS seeds are squares: x_{n+1} = x_n^2 mod M and the
    Blum-Goldwasser recall starts from x_0 = r^2 mod N.  Each y_j is
    the Q21 square of W(s, j)'s r, and -- Euler's criterion -- a quadratic
    residue modulo BOTH prime factors of its modulus (an oracle that stored r
    instead of r^2 would fail this for ~3/4 of the instances).  x = lo W(s,8),
    tp = lo W(s,9)."""
    mods, primes = _bbs_moduli_independent()
    st = O.init_states(O.V2, seed, 4096, 64)
    n_r_not_qr = 0
    for row, s in zip(st, range(4096, 4160)):
        for j in range(8):
            y_exp, mi, r = _q21_seed(O.splitmix_word(seed, s, j), mods)
            assert int(row[j]) == y_exp and int(row[8 + j]) == mi
            M = mods[mi]
            for p in (p for p in primes if M % p == 0):
                assert pow(int(row[j]), (p - 1) // 2, p) == 1          # Euler: QR mod p
                n_r_not_qr += pow(r, (p - 1) // 2, p) != 1
        assert int(row[16]) == O.splitmix_word(seed, s, 8) & M32
        assert int(row[17]) == O.splitmix_word(seed, s, 9) & M32
    assert n_r_not_qr > 100        # the criterion does discriminate r from r^2


def test_v2_seed_rejection_loop_injected():
    """Q21's rejection steps, reached by injected words: r landing on a prime
    factor of M (gcd != 1) and on a non-trivial square root of 1 (r^2 = 1
    mod M, found by CRT) both step to the next admissible r (for the root r + 1 = 40 * 251 is
    rejected too, so it steps twice)."""
    mods, primes = _bbs_moduli_independent()
    mi = 77
    M = mods[mi]                       # 239 * 251 = 59989
    p, q = 239, 251
    assert p * q == M
    # non-trivial root of 1: r = 1 (mod p), r = -1 (mod q)
    root = next(r for r in range(2, M - 1) if r % p == 1 and r % q == q - 1)
    assert pow(root, 2, M) == 1
    assert root == 10039 and (root + 1) % q == 0   # so the root steps twice
    for r0, r_expect in ((p, p + 1), (2 * q, 2 * q + 1), (root, root + 2)):
        w = (mi << 32) | (r0 - 2)     # 2 + lo mod (M - 3) = r0
        st = O.init_from_words(O.V2, [w] * 8 + [0, 0])
        assert [int(v) for v in st[:8]] == [pow(r_expect, 2, M)] * 8
        assert [int(v) for v in st[8:16]] == [mi] * 8
        assert _q21_seed(w, mods)[2] == r_expect
