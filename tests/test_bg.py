"""Blum-Goldwasser and the chaotic variant -- oracle
pins, not gpu: the hand-derived worked examples (tests/golden/bg_examples.json,
P:1327-1386), closed forms checked with Python's own big-integer pow, and
exhaustive round trips over small keys (SPEC's invariants)."""
import math

import numpy as np
import pytest

import oracle as O
import workloads as W


def test_worked_examples(golden):
    e = golden["bg_examples"]
    assert O.modpow(e["modpow"]["a"], e["modpow"]["e"], e["modpow"]["m"]) == e["modpow"]["value"]
    assert O.modinv(e["modinv"]["a"], e["modinv"]["m"]) == e["modinv"]["value"]
    c = e["classic"]
    ct, y = O.cbg_encrypt(False, c["N"], 0, c["r"], c["m"])
    assert ct.tolist() == c["c"] and y == c["y"]
    assert O.cbg_decrypt(False, c["p"], c["q"], 0, c["c"], c["y"]).tolist() == e["classic_decrypt"]["m"]
    h = e["chaotic"]
    assert O.bg_unit_bits(h["N"]) == h["Nb"]
    ct, y = O.cbg_encrypt(True, h["N"], h["S0"], h["r"], h["m"])
    assert ct.tolist() == h["c"] and y == h["y"]
    assert O.cbg_decrypt(True, 7, 11, h["S0"], h["c"], h["y"]).tolist() == h["m"]


def test_unit_bits_closed_form():
    """Nb = floor(log2(log2 N)), against floating-point logs away from
    the thresholds N = 2^(2^t), and exactly at them."""
    for N in [3, 5, 15, 16, 17, 77, 255, 256, 257, 65535, 65536, 2**32 - 1, 2**32, 2**62 + 1]:
        want = max(0, math.floor(math.log2(math.log2(N)) + 1e-12))
        assert O.bg_unit_bits(N) == want, N


@pytest.mark.parametrize("bits", [16, 31])
def test_y_and_keystream_against_pow(bits):
    """y = x0^(2^L) mod N and x_i = r^(2^(i+1)) mod N, with Python's
    pow as the independent big-integer routine; the chaotic ciphertext is the
    cumulative-XOR (Eq. Oplus) construction over those x_i."""
    gen = W.rng(77 + bits)
    for p, q, N in W.bg_keys(gen, 4, bits):
        r = int(gen.integers(2, N - 1))
        while math.gcd(r, N) != 1:
            r += 1
        L = 37
        m = gen.integers(0, 256, L).astype(np.uint8)
        S0 = int(gen.integers(0, 2**O.bg_unit_bits(N)))
        c, y = O.cbg_encrypt(True, N, S0, r, m)
        assert y == pow(r, 2 ** (L + 1), N)
        nb = O.bg_unit_bits(N)
        B = 0
        for i in range(L):
            B ^= pow(r, 2 ** (i + 1), N) % 2**nb
            assert int(c[i]) == (int(m[i]) ^ B ^ S0) % 2**nb
        cc, yy = O.cbg_encrypt(False, N, 0, r, m & 1)
        assert yy == y and [int(v) for v in cc] == [(int(m[i]) ^ pow(r, 2 ** (i + 1), N)) & 1 for i in range(L)]


@pytest.mark.parametrize("p,q", [(7, 11), (11, 19), (19, 23)])
def test_round_trip_exhaustive_small(p, q):
    """decrypt(encrypt(m)) == m for every coprime r and every message of up to
    3 units (all S0 for the variant) -- SPEC's exhaustive invariant."""
    N = p * q
    nb = O.bg_unit_bits(N)
    rs = [r for r in range(1, N + 1) if math.gcd(r, N) == 1]
    for L in range(0, 4):
        msgs = [[(k >> (nb * i)) % 2**nb for i in range(L)] for k in range(2 ** (nb * L))]
        for r in rs[:: max(1, len(rs) // 12)]:
            for S0 in range(2**nb):
                for m in msgs:
                    c, y = O.cbg_encrypt(True, N, S0, r, m)
                    assert O.cbg_decrypt(True, p, q, S0, c, y).tolist() == m
            for m in msgs:
                mb = [v & 1 for v in m]
                c, y = O.cbg_encrypt(False, N, 0, r, mb)
                assert O.cbg_decrypt(False, p, q, 0, c, y).tolist() == mb


def test_invalid_keys_rejected():
    with pytest.raises(O.OracleError):
        O.cbg_encrypt(True, 77, 0, 7, [1, 2])  # gcd(r, N) = 7 would leak a factor
    with pytest.raises(O.OracleError):
        O.cbg_encrypt(True, 78, 0, 5, [1])  # even N
    with pytest.raises(O.OracleError):
        O.cbg_decrypt(True, 5, 11, 0, [1], 3)  # 5 is not 3 mod 4
