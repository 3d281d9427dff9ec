"""Statistical battery -- not gpu.

Pins: the oracle's integer counts against an independent numpy brute force
(np.unpackbits on tiny inputs, reading Q31's MSB-first bit order) and closed
forms of degenerate streams; the host p-value arithmetic against NIST SP
800-22's printed worked examples (tests/golden/nist_sp800_22_examples.json);
the whole count -> p-value pipeline against a true-uniform stub (SPEC: the
battery's p-values on uniform input are themselves uniform) and the SPEC
negative controls."""
import math

import numpy as np
import pytest

import oracle as O
import workloads as W
from paper_1112_5239_b200 import battery as B


def _bits(words: np.ndarray) -> np.ndarray:
    """(S, n) u32 -> (S, 32 n) bits, each word most significant bit first."""
    be = words.astype(">u4").view(np.uint8).reshape(words.shape[0], -1)
    return np.unpackbits(be, axis=1).astype(np.int64)


def _brute(words: np.ndarray) -> np.ndarray:
    S, n = words.shape
    b = _bits(words)
    st = np.zeros(264, np.uint64)
    st[0] = b.sum()
    st[1] = (b[:, 1:] != b[:, :-1]).sum()
    st[2] = ((b[:, 1:] == 1) & (b[:, :-1] == 1)).sum()
    st[3] = (b[:, 8:] != b[:, :-8]).sum()
    nb = n // 4
    if nb:
        blk = b[:, : nb * 128].reshape(S, nb, 128).sum(axis=2)
        st[4] = ((blk - 64) ** 2).sum()
        st[5] = S * nb
    st[6] = b[:, 0].sum()
    st[7] = b[:, -1].sum()
    for sh in (0, 8, 16, 24):
        st[8:] += np.bincount(((words >> sh) & 0xFF).ravel(), minlength=256).astype(np.uint64)
    return st


@pytest.mark.parametrize("shape", [(1, 1), (3, 9), (5, 12), (2, 33)])
def test_oracle_battery_brute_force(shape):
    words = W.random_words(W.rng(40 + shape[1]), shape)
    assert np.array_equal(O.battery(words), _brute(words))


def test_oracle_battery_closed_forms():
    S, n = 3, 8
    z = O.battery(np.zeros((S, n), np.uint32))
    assert z[:8].tolist() == [0, 0, 0, 0, S * (n // 4) * 64 * 64, S * (n // 4), 0, 0] and z[8] == 4 * S * n
    f = O.battery(np.full((S, n), 0xFFFFFFFF, np.uint32))
    assert f[:8].tolist() == [32 * S * n, 0, S * (32 * n - 1), 0, S * 2 * 4096, S * 2, S, S] and f[8 + 255] == 4 * S * n
    a = O.battery(np.full((S, n), 0x55555555, np.uint32))  # 0101...: every adjacent pair differs
    assert a[0] == 16 * S * n and a[1] == S * (32 * n - 1) and a[2] == 0 and a[3] == 0 and a[4] == 0
    h = O.battery(np.full((S, n), 0x00FF00FF, np.uint32))  # bytes alternate 00/FF: every lag-8 pair differs
    assert h[3] == S * (32 * n - 8)


def test_nist_examples_pin_pvalue_arithmetic(golden):
    e = golden["nist_sp800_22_examples"]
    m = e["frequency_monobit"]
    bits = [int(c) for c in m["bits"]]
    assert abs((2 * sum(bits) - len(bits)) / math.sqrt(len(bits)) - m["s_obs"]) < 1e-9
    assert abs(B.monobit_p(len(bits), sum(bits)) - m["p"]) < 1e-6
    bf = e["block_frequency"]
    bits = [int(c) for c in bf["bits"]]
    M = bf["M"]
    blocks = [sum(bits[i : i + M]) for i in range(0, len(bits) - M + 1, M)]
    ssd = sum((c - M / 2) ** 2 for c in blocks)
    assert abs(4 * ssd / M - bf["chi2"]) < 1e-12
    assert abs(B.block_frequency_p(M, len(blocks), ssd) - bf["p"]) < 1e-6
    se = e["serial"]
    n = se["n"]
    assert abs(B.psi_sq(se["counts3"], n) - se["psi3"]) < 1e-9
    assert abs(B.psi_sq(se["counts2"], n) - se["psi2"]) < 1e-9
    assert abs(B.psi_sq(se["counts1"], n) - se["psi1"]) < 1e-9
    d1 = se["psi3"] - se["psi2"]
    d2 = se["psi3"] - 2 * se["psi2"] + se["psi1"]
    assert abs(B.igamc(2 ** (3 - 2), d1 / 2) - se["p1"]) < 1e-6
    assert abs(B.igamc(2 ** (3 - 3), d2 / 2) - se["p2"]) < 1e-6


def test_uniform_stub_pvalues_are_uniform():
    """SPEC (stat-stream invariants): on a true-uniform stub (numpy PCG64) the
    battery's p-values over 200 sub-streams are themselves uniform (KS, alpha
    0.001) -- this exercises the counts -> p-value pipeline, including the
    transition-form runs test and the serial statistic (readings Q31, Q32)."""
    from scipy.stats import kstest

    gen = np.random.default_rng(2024)
    S, n = 16, 256
    ps = {}
    for _ in range(200):
        words = gen.integers(0, 2**32, size=(S, n), dtype=np.uint64).astype(np.uint32)
        for k, v in B.pvalues(O.battery(words), S, n).items():
            ps.setdefault(k, []).append(v)
    for k, v in ps.items():
        assert kstest(v, "uniform").pvalue > 1e-3, k


def test_negative_controls():
    """an all-zero stream fails monobit; strictly alternating bits
    fail the runs test."""
    S, n = 4, 64
    p = B.pvalues(O.battery(np.zeros((S, n), np.uint32)), S, n)
    assert p["monobit"] < 1e-100 and not B.passes(p)
    p = B.pvalues(O.battery(np.full((S, n), 0x55555555, np.uint32)), S, n)
    assert p["runs"] < 1e-100 and not B.passes(p)


@pytest.mark.parametrize("variant", [O.V0, O.V1, O.V2, O.V3, O.V4])
def test_oracle_streams_pass_battery(variant):
    S, n = 64, 2048
    out = O.generate(variant, O.init_states(variant, W.SEEDS[0], 0, S), n)
    assert B.passes(B.pvalues(O.battery(out), S, n), alpha=1e-4)
