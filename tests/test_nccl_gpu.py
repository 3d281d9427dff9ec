"""The a7 row on a real GPU: consumer statistics all-reduced over the NCCL
process group (torchrun, one process per GPU; one GPU here, so world size 1
exercises the NCCL path end to end), equal to the oracle's statistics of
the same stream space."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("variant", [1, 2])
def test_torchrun_nccl_consume_matches_oracle(variant):
    S, n, calls = 2048, 64, 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "tools", "dist_consume.py"),
           "--streams", str(S), "--rounds", str(n), "--calls", str(calls), "--variant", str(variant)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    got = json.loads(line)["stats"]
    st = O.init_states(variant, json.loads(line).get("seed", 0x0123456789ABCDEF), 0, S)
    ref = np.zeros(258, np.uint64)
    for _ in range(calls):
        O.stats(O.generate(variant, st, n), ref)
    assert got == [int(v) for v in ref]
