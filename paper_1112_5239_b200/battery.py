"""Host-side p-values of the on-device statistical battery (SURVEY s8(f)
NEXT-2; monobit frequency, block frequency m = 128, runs,
serial 2-bit, byte chi-square, 8-lag autocorrelation -- the desk-scale
stand-in for the BigCrush runs of PAPER.md P:851-853).

The device (``ChaoticPRNG.battery``, C-ABI ``prng_battery``) returns integer
counts only; this module turns them into two-sided p-values.  Bit sequence
(reading Q31): each stream's words within one call, in round order, most
significant bit first; sequences never continue across streams or calls.
With S streams of N = 32 n bits:

* monobit: S_obs = |2 ones - S N| / sqrt(S N), p = erfc(S_obs / sqrt 2)
  (NIST SP 800-22 s2.1);
* block frequency, M = 128 (4 words): chi^2 = 4 M sum (pi_i - 1/2)^2 =
  sum (c_i - 64)^2 / 32 over the blocks, p = igamc(blocks / 2, chi^2 / 2)
  (NIST s2.2);
* runs, in transition form (reading Q32): for independent uniform bits the
  indicators [e_j != e_{j+1}] are themselves i.i.d. fair, so the number of
  differing adjacent pairs D ~ Binomial(S (N - 1), 1/2) exactly; z-test.
  NIST's s2.3 statistic is not used because its large-n mean 2 n pi (1 - pi)
  drops the +1/2 per sequence, an O(S) bias that is many standard
  deviations once S ~ 10^6 sequences are aggregated;
* 8-lag autocorrelation: likewise [e_j != e_{j+8}] are i.i.d. fair, so
  A ~ Binomial(S (N - 8), 1/2); z-test;
* serial, m = 2 (NIST s2.11 statistics without the wrap-around): pattern
  counts of the S (N - 1) overlapping pairs, c01 - c10 = last - first ones;
  psi2_m = 2^m / n sum c^2 - n, del psi2 = psi2_2 - psi2_1(first bits)
  ~ chi^2(2), del2 psi2 = psi2_2 - psi2_1(first) - psi2_1(second) ~ chi^2(1)
  (NIST's psi2_2 - 2 psi2_1 + psi2_0 when the counts wrap around), all with
  n = S (N - 1) pairs;
* byte chi-square: 256 bins over all four bytes of every word, 255 df.
"""
from __future__ import annotations

import math

import numpy as np

try:  # regularised upper incomplete gamma
    from scipy.special import gammaincc as _igamc
except Exception:  # pragma: no cover - scipy is in the image
    _igamc = None


def igamc(a: float, x: float) -> float:
    """Q(a, x) = Gamma(a, x) / Gamma(a) (NIST's igamc)."""
    if _igamc is None:
        raise RuntimeError("scipy.special.gammaincc unavailable")
    return float(_igamc(a, x))


def z_two_sided(z: float) -> float:
    return math.erfc(abs(z) / math.sqrt(2.0))


def monobit_p(n_bits: int, ones: int) -> float:
    return z_two_sided((2 * ones - n_bits) / math.sqrt(n_bits))


def block_frequency_p(M: int, blocks: int, sum_sq_dev: float) -> float:
    """sum_sq_dev = sum over blocks of (c_i - M/2)^2 (c_i ones in block i)."""
    chi2 = 4.0 * sum_sq_dev / M
    return igamc(blocks / 2.0, chi2 / 2.0)


def binomial_half_p(successes: int, trials: int) -> float:
    return z_two_sided((2 * successes - trials) / math.sqrt(trials))


def psi_sq(counts, n: int) -> float:
    """NIST psi^2_m from the 2^m pattern counts of n (overlapping) patterns."""
    m_pat = len(counts)
    return m_pat / n * float(sum(int(c) ** 2 for c in counts)) - n


def serial_p(c2: tuple[int, int, int, int], n: int) -> tuple[float, float]:
    """m = 2 over n overlapping pairs, c2 = (c00, c01, c10, c11).  Without
    NIST's wrap-around the first- and second-bit marginals differ slightly, so
    del psi2 uses the first-bit marginal (the 2-df Markov statistic) and
    del2 psi2 = psi2_2 - psi2_1(first) - psi2_1(second) (the 1-df independence
    statistic, >= 0); both reduce to NIST's with circular counts."""
    c00, c01, c10, c11 = c2
    first = (c00 + c01, c10 + c11)
    second = (c00 + c10, c01 + c11)
    p2 = psi_sq(c2, n)
    d1 = p2 - psi_sq(first, n)
    d2 = max(0.0, p2 - psi_sq(first, n) - psi_sq(second, n))
    return igamc(1.0, d1 / 2.0), igamc(0.5, d2 / 2.0)


def chi2_uniform_p(hist) -> float:
    h = np.asarray(hist, dtype=np.float64)
    e = h.sum() / len(h)
    chi2 = float(((h - e) ** 2).sum() / e)
    return igamc((len(h) - 1) / 2.0, chi2 / 2.0)


def pvalues(stats, n_streams: int, n: int) -> dict:
    """p-values of one battery block (or several calls' blocks of the same
    shape accumulated: pass n_streams * calls)."""
    s = [int(v) for v in np.asarray(stats, dtype=np.uint64)[:8]]
    ones, diff, c11, lag8, bsq, blocks, first, last = s
    N = 32 * n
    bits = n_streams * N
    pairs = n_streams * (N - 1)
    c01 = (diff + last - first) // 2
    c10 = diff - c01
    c00 = pairs - diff - c11
    p_ser1, p_ser2 = serial_p((c00, c01, c10, c11), pairs)
    out = {
        "monobit": monobit_p(bits, ones),
        "runs": binomial_half_p(diff, pairs),
        "autocorrelation_lag8": binomial_half_p(lag8, n_streams * (N - 8)),
        "serial_2bit": p_ser1,
        "serial_2bit_del2": p_ser2,
        "byte_chi2": chi2_uniform_p(np.asarray(stats, dtype=np.uint64)[8:264]),
    }
    if blocks:
        out["block_frequency_128"] = block_frequency_p(128, blocks, bsq)
    return out


def passes(p: dict, alpha: float = 1e-4) -> bool:
    return all(alpha < v < 1 - alpha for v in p.values())
