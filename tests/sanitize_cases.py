"""Small-shape run of every kernel family, for compute-sanitizer
(tests/test_sanitizers_gpu.py; VERDICT r1 "sanitizer evidence").

Each case goes through the C-ABI and is also checked word for word against
the oracle, so a run under memcheck / racecheck / synccheck / initcheck both
exercises the shared-memory and async-proxy (TMA) paths and proves they still
produce the right words.  Shapes are tiny (a few tiles plus a ragged tail):
the sanitizers slow kernels down by 10-1000x.

Store paths covered (csrc/api.cu run_pass):
  * 2-D TMA boxes (V1 n = 128, V3 n = 128; any n % 4 == 0 with aligned rows),
    16- and 8-round boxes, 1 and 3 buffers
  * 3-D band boxes (V1 n = 256)
  * staged shared-memory + coalesced STG (V1 / V3 n % 4 != 0; misaligned output)
  * direct 128-bit / scalar stores (STORE_DIRECT; V0, V2, V4)
  * the single-stream V0 jump-ahead kernel (C1)
plus the fused consumer (V0..V4), the battery, generate_host, the digest,
chaotic Blum-Goldwasser encrypt / decrypt, Algorithm 1 and the Gamma(f) check.

    python tests/sanitize_cases.py [case ...]     (default: all)
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_1112_5239_b200 as P  # noqa: E402

SEED = 0x0123456789ABCDEF
S = 32 * 7  # 3.5 fast tiles of 64 streams: a partial last tile


def _gen(variant, n, *, env=None, store_path=P.STORE_AUTO, offset=0, S_=S):
    old = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        g = P.ChaoticPRNG(SEED, S_, variant, store_path=store_path)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    st = O.init_states(variant, SEED, 0, S_)
    for _ in range(2):  # two calls: state carry (and V2 rotation)
        buf = torch.empty(S_ * n + offset, dtype=torch.int32, device="cuda")
        view = buf[offset:]
        g.generate(n, out=view)
        got = P.as_u32(view).reshape(S_, n)
        ref = O.generate(variant, st, n)
        assert np.array_equal(got, ref), f"V{variant} n={n} env={env} path={store_path} offset={offset}"
    assert np.array_equal(g.get_state(), O.state_planes(variant, st))
    g.close()


def case_tma2d():
    _gen(P.V1, 128)
    _gen(P.V1, 128, env={"CIPRNG_V1_COLS": "16"})
    _gen(P.V1, 128, env={"CIPRNG_V1_COLS": "8"})
    _gen(P.V1, 128, env={"CIPRNG_V1_COLS": "32", "CIPRNG_V1_BUFS": "1"})
    _gen(P.V1, 128, env={"CIPRNG_V1_COLS": "32", "CIPRNG_V1_BUFS": "3"})
    _gen(P.V3, 128)


def case_band3d():
    _gen(P.V1, 256)
    _gen(P.V1, 256, env={"CIPRNG_V1_COLS": "128"})
    _gen(P.V1, 256, env={"CIPRNG_V1_COLS": "64", "CIPRNG_V1_BUFS": "1"})


def case_staged():
    # no TMA descriptor when n % 4 != 0 or the rows are not 16-byte aligned
    _gen(P.V1, 37)
    _gen(P.V1, 38)
    _gen(P.V1, 128, offset=1)
    _gen(P.V3, 37)
    _gen(P.V1, 128, env={"CIPRNG_V1_SMEM_STG": "1"}, store_path=P.STORE_DIRECT)


def case_direct():
    for v, n in ((P.V1, 128), (P.V1, 5), (P.V3, 64), (P.V0, 20), (P.V2, 16), (P.V4, 20)):
        _gen(v, n, store_path=P.STORE_DIRECT)
    _gen(P.V2, 17)


def case_jump():
    # one V0 stream split over the GPU (csrc/v0_jump.cu: shared-memory windows,
    # block scans, cooperative look-back); 3 CTAs of 128 segments x 16 rounds
    for n in (5000, 4096):
        _gen(P.V0, n, S_=1)
    _gen(P.V0, 5000, S_=3)  # three streams: three CTA rows, separate look-backs
    g = P.ChaoticPRNG(0, 1, P.V0, paper_defaults=True)
    st = O.init_states(P.V0, 0, 0, 1, paper_defaults=True)
    got = P.as_u32(g.generate(6000))
    assert np.array_equal(got, O.generate(P.V0, st, 6000)), "jump paper_defaults"
    assert int(g.info().store_path) == 3, "jump path not taken"
    g.close()


def case_consume():
    for v, n in ((P.V0, 20), (P.V1, 64), (P.V1, 66), (P.V2, 16), (P.V3, 64), (P.V4, 20)):
        g = P.ChaoticPRNG(SEED, S, v)
        got = P.as_u64(g.consume(n))
        ref = O.stats(O.generate(v, O.init_states(v, SEED, 0, S), n))
        assert np.array_equal(got, ref), f"consume V{v} n={n}"
        g.close()


def case_battery():
    for v, n in ((P.V1, 64), (P.V1, 6), (P.V2, 8), (P.V3, 64), (P.V0, 8)):
        g = P.ChaoticPRNG(SEED, S, v)
        got = P.as_u64(g.battery(n))
        ref = O.battery(O.generate(v, O.init_states(v, SEED, 0, S), n))
        assert np.array_equal(got, ref), f"battery V{v} n={n}"
        g.close()


def case_host():
    for v, n in ((P.V1, 128), (P.V1, 36), (P.V2, 16)):
        g = P.ChaoticPRNG(SEED, S, v)
        got = g.generate_host(n).numpy().view(np.uint32)
        assert np.array_equal(got, O.generate(v, O.init_states(v, SEED, 0, S), n)), f"host V{v}"
        g.close()


def case_digest():
    # direct stores: initcheck does not see TMA (async-proxy) writes
    g = P.ChaoticPRNG(SEED, S, P.V1, store_path=P.STORE_DIRECT)
    out = g.generate(64)
    # accumulator initialised by a host copy (initcheck tracks copies; a torch
    # fill kernel is outside the --kernel-name filter and would not count)
    acc = torch.tensor([0], dtype=torch.int64, device="cuda")
    d = int(P.as_u64(P.digest(out, 5, acc))[0])
    ref = int(O.digest(P.as_u32(out), 5))
    assert d == ref, "digest"
    g.close()


def case_bg():
    from paper_1112_5239_b200 import bg as BG

    for chaotic in (False, True):
        m = torch.tensor([[2, 3, 1, 0]], dtype=torch.uint8, device="cuda")
        N = torch.tensor([77], device="cuda")
        c, y = BG.encrypt(chaotic, N, torch.tensor([3], device="cuda"), m,
                          torch.tensor([1], dtype=torch.int32, device="cuda"))
        rc, ry = O.cbg_encrypt(chaotic, 77, 1, 3, [2, 3, 1, 0])
        assert c.cpu().numpy()[0].tolist() == rc.tolist() and int(y.item()) == ry, "cbg encrypt"
        back = BG.decrypt(chaotic, torch.tensor([7], device="cuda"), torch.tensor([11], device="cuda"), c, y,
                          torch.tensor([1], dtype=torch.int32, device="cuda"))
        mm, status = back
        ref = O.cbg_decrypt(chaotic, 7, 11, 1, rc, ry).tolist()  # units of 1 bit unless chaotic
        assert mm.cpu().numpy()[0].tolist() == ref and int(status[0]) == 0, "cbg decrypt"


def case_chaos():
    from paper_1112_5239_b200 import chaos as CH

    z0 = np.array([1, 7, 12345, 99, 3], np.uint32)
    z = torch.tensor(z0.view(np.int32), device="cuda")
    x = torch.zeros(5, dtype=torch.int32, device="cuda")
    got = CH.alg1_generate(8, 4, z, x, 5).cpu().numpy().view(np.uint32)
    assert np.array_equal(got, O.alg1_generate(None, 8, 4, z0, np.zeros(5, np.uint32), 5)), "alg1"
    assert CH.gamma_check(6)["chaotic"], "gamma"


CASES = {k[5:]: v for k, v in globals().items() if k.startswith("case_")}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    torch.cuda.set_device(0)
    import time

    for name in names:
        t0 = time.time()
        CASES[name]()
        torch.cuda.synchronize()
        print(f"case {name} ok ({time.time() - t0:.1f} s)", flush=True)
    print("sanitize cases ok")
