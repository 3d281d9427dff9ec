"""GPU batch Blum-Goldwasser / chaotic variant against
the oracle, byte for byte: many independent messages per launch, small and
~2^62 moduli, L spanning the 16-unit vector path and its ragged tail, L = 0,
invalid keys; then decryption round trips on the GPU."""
import math

import numpy as np
import pytest
import torch

import oracle as O
import workloads as W
from paper_1112_5239_b200 import bg as BG

pytestmark = pytest.mark.gpu


def _batch(gen, B, bits):
    keys = W.bg_keys(gen, B, bits) if bits > 4 else [(7, 11, 77)] * B
    rs, S0s = [], []
    for p, q, N in keys:
        r = int(gen.integers(1, N))
        while math.gcd(r, N) != 1:
            r = r % (N - 1) + 1
        rs.append(r)
        S0s.append(int(gen.integers(0, 2 ** O.bg_unit_bits(N))))
    return keys, rs, S0s


def _t64(v):
    return torch.tensor(np.array(v, dtype=np.uint64).view(np.int64), device="cuda")


@pytest.mark.parametrize("chaotic", [True, False])
@pytest.mark.parametrize("bits,L", [(4, 3), (16, 17), (31, 0), (31, 1), (31, 16), (31, 100), (20, 1024)])
def test_cbg_encrypt_decrypt_matches_oracle(chaotic, bits, L):
    gen = W.rng(500 + bits + L)
    B = 96
    keys, rs, S0s = _batch(gen, B, bits)
    m = gen.integers(0, 256, (B, L)).astype(np.uint8)
    N = _t64([k[2] for k in keys])
    S0 = torch.tensor(S0s, dtype=torch.int32, device="cuda")
    c, y = BG.encrypt(chaotic, N, _t64(rs), torch.from_numpy(m).cuda(), S0)
    c, y = c.cpu().numpy(), y.cpu().numpy().view(np.uint64)
    for k, (p, q, Nk) in enumerate(keys):
        rc, ry = O.cbg_encrypt(chaotic, Nk, S0s[k], rs[k], m[k])
        assert np.array_equal(c[k], rc) and int(y[k]) == ry, k
    mm, st = BG.decrypt(chaotic, _t64([k[0] for k in keys]), _t64([k[1] for k in keys]), torch.from_numpy(c).cuda(),
                        _t64(y), S0)
    mask = 2 ** np.array([O.bg_unit_bits(k[2]) if chaotic else 1 for k in keys], dtype=np.uint16)[:, None] - 1
    assert (st.cpu().numpy() == 0).all()
    assert np.array_equal(mm.cpu().numpy(), (m & mask).astype(np.uint8))


def test_cbg_invalid_inputs_flagged():
    N = _t64([77, 78, 77, 2**63 + 1])
    r = _t64([3, 5, 7, 3])  # gcd(7, 77) = 7; 78 even; N >= 2^63
    m = torch.zeros((4, 8), dtype=torch.uint8, device="cuda")
    _, y = BG.encrypt(True, N, r, m)
    assert y.cpu().tolist()[1:] == [0, 0, 0] and y.cpu().tolist()[0] == O.cbg_encrypt(True, 77, 0, 3, [0] * 8)[1]
    _, st = BG.decrypt(True, _t64([7, 5]), _t64([11, 11]), torch.zeros((2, 4), dtype=torch.uint8, device="cuda"),
                       _t64([25, 3]))
    assert st.cpu().tolist() == [0, 1]
