"""Algorithm 1 and the Gamma(f) checks -- oracle pins,
not gpu.  Theorem 1 / Theorem 2 special cases the
paper and SPEC state (vectorial negation satisfies both; identity
and constant functions do not), an independent Kosaraju SCC count against the
reachability form, the SPEC's hand-derived arcs of f = [3,2,1,0], and Alg. 1
against a hand trace and its iteration-count bounds."""
import numpy as np
import pytest

import oracle as O
import workloads as W


def _apply_single(f, n, i, x):
    fx = (~x & ((1 << n) - 1)) if f is None else int(f[x])
    bit = 1 << (i - 1)
    return (x & ~bit) | (fx & bit)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 10])
def test_negation_satisfies_both_theorems(n):
    """'the vectorial negation satisfies the hypotheses of both
    theorems' -- Gamma is the hypercube (strongly connected, every vertex has
    in = out = n)."""
    r = O.gamma_reach(None, n)
    assert r.tolist() == [2**n, 2**n, 0]
    c = O.gamma_check(None, n)
    assert c == {"scc": 1, "doubly_stochastic": True, "unbalanced": 0}


def test_identity_and_constant():
    """identity -> 2^n singleton components (not chaotic, M = I
    doubly stochastic); constant 0 -> not chaotic, not doubly stochastic."""
    n = 4
    ident = np.arange(2**n, dtype=np.uint32)
    assert O.gamma_check(ident, n) == {"scc": 2**n, "doubly_stochastic": True, "unbalanced": 0}
    assert O.gamma_reach(ident, n).tolist() == [1, 1, 0]
    z = np.zeros(4, np.uint32)
    c = O.gamma_check(z, 2)
    assert c["scc"] == 4 and not c["doubly_stochastic"]
    # from 00 nothing but 00 is reachable; every vertex reaches 00 by clearing bits
    assert O.gamma_reach(z, 2).tolist()[:2] == [1, 4]


def test_table_negation_arcs_hand():
    """f = [3,2,1,0] (n = 2) -- from 00 the arcs go to 01 (cell 1)
    and 10 (cell 2); the same graph as the built-in negation."""
    f = np.array([3, 2, 1, 0], np.uint32)
    assert _apply_single(f, 2, 1, 0) == 1 and _apply_single(f, 2, 2, 0) == 2
    assert O.gamma_reach(f, 2).tolist() == O.gamma_reach(None, 2).tolist()


@pytest.mark.parametrize("seed", range(12))
def test_reachability_form_matches_scc_count(seed):
    """Strongly connected (Kosaraju count == 1) iff both reachability counts are
    2^n; degree balance identical in both oracle routines."""
    gen = W.rng(300 + seed)
    n = int(gen.integers(2, 7))
    # mix of random tables and perturbed negations (some chaotic, some not)
    f = gen.integers(0, 2**n, 2**n).astype(np.uint32)
    if seed % 2:
        f = (~np.arange(2**n, dtype=np.uint32)) & (2**n - 1)
        f[int(gen.integers(0, 2**n))] ^= 1 << int(gen.integers(0, n))
        f = f.astype(np.uint32)
    c, r = O.gamma_check(f, n), O.gamma_reach(f, n)
    assert (c["scc"] == 1) == (int(r[0]) == 2**n and int(r[1]) == 2**n)
    assert c["unbalanced"] == int(r[2])


def test_alg1_hand_trace():
    """Alg. 1 with f = negation, n = 4, b = 1, z = 1 (Q34): the
    xorshift32 sequence from 1 is 270369, 67634689, 2647435461, ... (Alg. 2;
    270369 is SPEC S:54's worked value) so k = 1 + (1 + 270369 % 1) = 2 and
    the cells are 1 + 67634689 % 4 = 2, 1 + 2647435461 % 4 = 2,
    1 + 307599695 % 4 = 4: x = 0 -> 0b0010 -> 0 -> 0b1000."""
    assert O.xorshift32_seq(1, 4) == [270369, 67634689, 2647435461, 307599695]
    z = np.array([1], np.uint32)
    x = np.array([0], np.uint32)
    out = O.alg1_generate(None, 4, 1, z, x, 1)
    assert out.tolist() == [[0b1000]]


def test_alg1_iteration_count_bounds():
    """k + 1 in [b + 2, 2b + 1] single-cell updates per output (P:444-446 and
    SPEC's off-by-one note): with f = negation each update flips one bit, so
    popcount parity of consecutive outputs follows the update count; check the
    count itself by replaying the draws."""
    b, n = 8, 6
    z0 = 123456789
    z = np.array([z0], np.uint32)
    x = np.array([0], np.uint32)
    out = O.alg1_generate(None, n, b, z, x, 200)[0]
    seq = O.xorshift32_seq(z0, 200 * (2 * b + 2))
    pos, xv = 0, 0
    for j in range(200):
        k = b + 1 + seq[pos] % b
        pos += 1
        assert b + 2 <= k + 1 <= 2 * b + 1
        for _ in range(k + 1):
            xv ^= 1 << (seq[pos] % n)
            pos += 1
        assert int(out[j]) == xv
