"""GPU Algorithm 1 and Gamma(f) checks against the
oracle: bit-exact configurations for negation and table functions, in-place
state advance, and identical reachability / balance reports."""
import numpy as np
import pytest
import torch

import oracle as O
import workloads as W
from paper_1112_5239_b200 import chaos as C

pytestmark = pytest.mark.gpu


def _i32(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).cuda()


@pytest.mark.parametrize("n_out", [37, 64])  # ragged rows (scalar stores) / 8-word sector chunks
@pytest.mark.parametrize("n,b,table", [(4, 1, False), (16, 8, False), (32, 3, False), (4, 5, True), (12, 8, True),
                                       (16, 2, True), (6, 3, False)])
def test_alg1_matches_oracle(n, b, table, n_out):
    gen = W.rng(700 + n + b)
    S = 1000
    f = gen.integers(0, 2**n, 2**n).astype(np.uint32) if table else None
    z = gen.integers(1, 2**32, S).astype(np.uint32)
    x = (gen.integers(0, 2**32, S) & ((1 << n) - 1 if n < 32 else 0xFFFFFFFF)).astype(np.uint32)
    zt, xt = _i32(z), _i32(x)
    got = C.alg1_generate(n, b, zt, xt, n_out, f=None if f is None else _i32(f))
    zr, xr = z.copy(), x.copy()
    ref = O.alg1_generate(f, n, b, zr, xr, n_out)
    assert np.array_equal(got.cpu().numpy().view(np.uint32), ref)
    assert np.array_equal(zt.cpu().numpy().view(np.uint32), zr)
    assert np.array_equal(xt.cpu().numpy().view(np.uint32), xr)


@pytest.mark.parametrize("case", ["negation", "identity", "constant", "random", "perturbed", "perm"])
@pytest.mark.parametrize("n", [2, 6, 11, 16])
def test_gamma_check_matches_oracle(case, n):
    gen = W.rng(800 + n)
    V = 2**n
    if case == "negation":
        f = None
    elif case == "identity":
        f = np.arange(V, dtype=np.uint32)
    elif case == "constant":
        f = np.zeros(V, np.uint32)
    elif case == "random":
        f = gen.integers(0, V, V).astype(np.uint32)
    elif case == "perturbed":
        f = (~np.arange(V, dtype=np.uint32)) & (V - 1)
        f[gen.integers(0, V, 3)] ^= 1
        f = f.astype(np.uint32)
    else:
        f = gen.permutation(V).astype(np.uint32)
    got = C.gamma_check(n, None if f is None else _i32(f))
    ref = O.gamma_reach(f, n)
    assert [got["reach_from_0"], got["reach_to_0"], got["unbalanced"]] == ref.tolist()
    if case == "negation":
        assert got["chaotic"] and got["doubly_stochastic"]


def test_theorem2_uniformity_by_sampling():
    """Theorem 2 observed on the GPU: with Gamma(f) strongly
    connected, Algorithm 1's outputs tend to the uniform law iff M is doubly
    stochastic.  f = negation (doubly stochastic) gives a uniform histogram
    over the 2^n configurations; a negation with one flipped table bit that
    stays strongly connected but loses the degree balance (checked by the
    oracle) gives a grossly non-uniform one."""
    from scipy.stats import chisquare

    n, V = 6, 64
    gen = W.rng(900)
    f_bad = ((~np.arange(V, dtype=np.uint32)) & (V - 1)).astype(np.uint32)
    f_bad[int(gen.integers(0, V))] ^= 1 << int(gen.integers(0, n))
    r = O.gamma_reach(f_bad, n)
    assert int(r[0]) == V and int(r[1]) == V and int(r[2]) > 0  # chaotic, not doubly stochastic
    S, n_out = 2**16, 64
    p = {}
    for name, f in (("negation", None), ("unbalanced", f_bad)):
        z = _i32(gen.integers(1, 2**32, S).astype(np.uint32))
        x = _i32(gen.integers(0, V, S).astype(np.uint32))
        out = C.alg1_generate(n, 8, z, x, n_out, f=None if f is None else _i32(f))
        # after a burn-in, every 4th output (consecutive calls share x)
        hist = torch.bincount(out[:, 16::4].reshape(-1).long(), minlength=V).cpu().numpy()
        p[name] = chisquare(hist).pvalue
    assert p["negation"] > 1e-4 and p["unbalanced"] < 1e-12, p


def test_alg1_and_gamma_validate_arguments():
    """The kernels index z/x up to z.numel() - 1 and f up to 2^n - 1, so the
    binding rejects short, mistyped or non-contiguous tensors before launch."""
    z = torch.ones(64, dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError):
        C.alg1_generate(8, 4, z, torch.zeros(63, dtype=torch.int32, device="cuda"), 4)
    with pytest.raises(ValueError):
        C.alg1_generate(8, 4, z, torch.zeros(64, dtype=torch.int64, device="cuda"), 4)
    with pytest.raises(ValueError):
        C.alg1_generate(8, 4, z, torch.zeros(128, dtype=torch.int32, device="cuda")[::2], 4)
    with pytest.raises(ValueError):
        C.alg1_generate(8, 4, z, torch.zeros(64, dtype=torch.int32, device="cuda"), 4,
                         f=torch.zeros(255, dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError):
        C.gamma_check(6, f=torch.zeros(32, dtype=torch.int32, device="cuda"))
    assert C.gamma_check(4, f=torch.arange(16, dtype=torch.int32, device="cuda") ^ 15)["chaotic"]
