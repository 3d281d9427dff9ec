"""prng_emit (include/ciprng.h): the generated words
serialised to a file descriptor as raw little-endian u32, hex lines or bit
lines.  The expected bytes are built here from the words (numpy '<u4'
bytes, "%08x\\n", 32 '0'/'1' MSB first + "\\n") -- the SPEC's definitions --
and the words themselves are checked against the oracle."""
import os

import numpy as np
import pytest
import torch

import oracle as O
import paper_1112_5239_b200 as P
import workloads as W

pytestmark = pytest.mark.gpu
SEED = W.SEEDS[0]


def _serialise(words: np.ndarray, fmt: str) -> bytes:
    words = words.reshape(-1)
    if fmt == "raw-le32":
        return words.astype("<u4").tobytes()
    if fmt == "hex":
        return "".join(f"{int(w):08x}\n" for w in words).encode()
    return "".join(f"{int(w):032b}\n" for w in words).encode()


@pytest.mark.parametrize("fmt", ["raw-le32", "hex", "bits"])
@pytest.mark.parametrize("variant,n", [(W.V1, 128), (W.V1, 37), (W.V2, 16), (W.V0, 9)])
def test_emit_matches_oracle(tmp_path, fmt, variant, n):
    S = 256
    g = P.ChaoticPRNG(SEED, S, variant)
    st = O.init_states(variant, SEED, 0, S)
    path = tmp_path / "out.bin"
    for call in range(2):  # state carries across emit calls like generate
        wrote = g.emit(n, str(path), fmt)
        data = path.read_bytes()
        ref = O.generate(variant, st, n)
        assert wrote == len(data)
        assert data == _serialise(ref, fmt), f"call {call}"
    g.close()


def test_emit_known_words_layout(tmp_path):
    """SPEC S:648 'known 4-word sequence -> 16 exact bytes': one stream of a
    V0 paper_defaults generator, 4 words, byte layout spelled out."""
    g = P.ChaoticPRNG(0, 1, W.V0, paper_defaults=True)
    words = O.generate(W.V0, O.init_states(W.V0, 0, 0, 1, paper_defaults=True), 4).reshape(-1)
    path = tmp_path / "w.bin"
    assert g.emit(4, str(path)) == 16
    data = path.read_bytes()
    for k, w in enumerate(words):
        w = int(w)
        assert list(data[4 * k:4 * k + 4]) == [w & 255, (w >> 8) & 255, (w >> 16) & 255, w >> 24]
    g.close()


def test_emit_multi_chunk_hex_equals_generate(tmp_path):
    """More than two ~64 MiB chunks of hex text: the pinned double buffer,
    the format kernel at s_begin != 0 and the host write overlap."""
    n = 64
    rows = (64 << 20) // (n * 9) // 64 * 64
    S = 2 * rows + 96
    g1 = P.ChaoticPRNG(SEED, S, W.V1)
    g2 = P.ChaoticPRNG(SEED, S, W.V1)
    path = tmp_path / "big.txt"
    wrote = g1.emit(n, str(path), "hex")
    assert wrote == S * n * 9 == os.path.getsize(path)
    dev = P.as_u32(g2.generate(n))
    raw = np.frombuffer(path.read_bytes(), dtype=np.uint8).reshape(S * n, 9)
    assert (raw[:, 8] == ord("\n")).all()
    digits = raw[:, :8].astype(np.int64)
    vals = np.where(digits >= ord("a"), digits - ord("a") + 10, digits - ord("0"))
    words = (vals * (16 ** np.arange(7, -1, -1))).sum(axis=1).astype(np.uint32)
    assert np.array_equal(words.reshape(S, n), dev)
    assert np.array_equal(g1.get_state(), g2.get_state())
    g1.close()
    g2.close()


def test_emit_zero_and_errors(tmp_path):
    g = P.ChaoticPRNG(SEED, 64, W.V1)
    path = tmp_path / "z.bin"
    assert g.emit(0, str(path)) == 0 and path.read_bytes() == b""
    with pytest.raises(ValueError):
        g.emit(4, str(path), "octal")
    # a write failure (read-only descriptor): PRNG_EIO, and the state still
    # advanced by the whole call, exactly like generate()
    twin = P.ChaoticPRNG(SEED, 64, W.V1)
    fd = os.open(os.devnull, os.O_RDONLY)
    try:
        with pytest.raises(P.PrngError) as ei:
            g.emit(8, fd)
        assert ei.value.status == -7
    finally:
        os.close(fd)
    twin.generate(8)
    torch.cuda.synchronize()
    assert np.array_equal(g.get_state(), twin.get_state())
    g.close()
    twin.close()


def test_emit_cli_to_stdout():
    """python -m paper_1112_5239_b200 writes raw-le32 to standard output."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "paper_1112_5239_b200", "--variant", "1", "--streams", "64", "--n",
                        "8", "--calls", "2", "--seed", str(SEED)], capture_output=True, cwd=root, timeout=300)
    assert r.returncode == 0, r.stderr.decode()[-2000:]
    st = O.init_states(W.V1, SEED, 0, 64)
    ref = np.concatenate([O.generate(W.V1, st, 8).reshape(-1) for _ in range(2)])
    assert r.stdout == ref.astype("<u4").tobytes()


def test_emit_single_stream_jump_path(tmp_path):
    """prng_emit over the C1 jump-ahead path (one V0 stream, n >= 4096): the
    hex lines equal the oracle's sequential chain."""
    n = 5000
    g = P.ChaoticPRNG(SEED, 1, W.V0)
    path = tmp_path / "j.txt"
    assert g.emit(n, str(path), "hex") == 9 * n
    assert int(g.info().store_path) == 3
    ref = O.generate(W.V0, O.init_states(W.V0, SEED, 0, 1), n)
    assert path.read_bytes() == _serialise(ref, "hex")
    g.close()
