"""The C ABI from a plain C program on the GPU (tests/c_abi_check.c, "gpu"
mode): prng_create / prng_generate_host for V1, V2 and a single V0 stream
(the jump-ahead path), two calls each, word for word against the C oracle
linked into the same test binary."""
import subprocess

import pytest

from tests.test_abi import _build_c_check

pytestmark = pytest.mark.gpu


def test_c_abi_generate_matches_oracle(tmp_path):
    exe = _build_c_check(tmp_path)
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "C ABI OK gpu" in r.stdout
