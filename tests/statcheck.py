"""Cheap frequency / chi-square sanity checks (SURVEY s4 layer 5; SPEC.md
S:633-641 lists the battery this is a small subset of).  Used on oracle and
GPU output alike; a stand-in for the paper's BigCrush claims (P:851-853,
P:923-925), which need TestU01 (not available)."""
from __future__ import annotations

import math

import numpy as np
from scipy import special, stats


def monobit_p(words: np.ndarray) -> float:
    """Two-sided p-value of the total number of one bits."""
    w = np.ascontiguousarray(words, dtype=np.uint32).ravel()
    ones = int(np.unpackbits(w.view(np.uint8)).sum())
    nbits = w.size * 32
    z = (2 * ones - nbits) / math.sqrt(nbits)
    return float(special.erfc(abs(z) / math.sqrt(2)))


def byte_chi2_p(words: np.ndarray) -> float:
    """Chi-square (255 dof) of the byte histogram; returns the upper-tail p."""
    w = np.ascontiguousarray(words, dtype=np.uint32).ravel()
    counts = np.bincount(w.view(np.uint8), minlength=256).astype(np.float64)
    exp = counts.sum() / 256.0
    chi2 = float(((counts - exp) ** 2 / exp).sum())
    return float(stats.chi2.sf(chi2, 255))


def hist_chi2_p(hist: np.ndarray) -> float:
    """Upper-tail p of a 256-bin top-byte histogram."""
    h = np.asarray(hist, dtype=np.float64)
    exp = h.sum() / h.size
    chi2 = float(((h - exp) ** 2 / exp).sum())
    return float(stats.chi2.sf(chi2, h.size - 1))


def runs_p(words: np.ndarray) -> float:
    """NIST SP800-22 runs test on the bit sequence."""
    bits = np.unpackbits(np.ascontiguousarray(words, dtype=np.uint32).ravel().view(np.uint8)).astype(np.int8)
    n = bits.size
    pi = bits.mean()
    if abs(pi - 0.5) >= 2 / math.sqrt(n):
        return 0.0
    v = 1 + int(np.count_nonzero(bits[1:] != bits[:-1]))
    num = abs(v - 2 * n * pi * (1 - pi))
    den = 2 * math.sqrt(2 * n) * pi * (1 - pi)
    return float(special.erfc(num / den))


def pi_zscore(inside: int, pairs: int) -> float:
    p = math.pi / 4
    sigma = math.sqrt(p * (1 - p) / pairs)
    return (inside / pairs - p) / sigma


def battery(words: np.ndarray) -> dict:
    return {"monobit": monobit_p(words), "byte_chi2": byte_chi2_p(words), "runs": runs_p(words)}


def passes(ps: dict, alpha: float = 1e-4) -> bool:
    return all(alpha <= p <= 1 - alpha for p in ps.values()) if ps else False
