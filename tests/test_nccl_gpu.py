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


def test_bench_multi_rank_path_on_one_gpu():
    """bench.py's torchrun (N > 1) code path end to end: two ranks sharing the
    one GPU here over gloo (the driver's N-GPU runs use NCCL, one GPU each).
    Rank 0 alone prints one JSON line; the stream space is the union of both
    shards; timing is the max over ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "6", "--warmup", "3", "--streams", "65536", "--no-secondary", "--e2e-steps", "1"]
    env = dict(os.environ, CIPRNG_BENCH_BACKEND="gloo")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["global_streams"] == 2 * 65536 and d["value"] > 0
    assert d["scaling"] == "weak" and "cpu_baseline" not in d


def test_bench_c5_consume_allreduce_two_ranks():
    """bench.py's C5 row across ranks (consume + SUM all-reduce of the 258
    statistics per call, max-over-ranks timing): two ranks sharing the one
    GPU here over gloo.  The reduced counters cover the whole job exactly."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "4", "--warmup", "3", "--streams", "65536", "--c5-only", "--e2e-steps", "1"]
    env = dict(os.environ, CIPRNG_BENCH_BACKEND="gloo")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    c5 = d["secondary"]["c5_consume_allreduce"]
    assert c5["n_gpus"] == 2 and c5["global_streams"] == 2 * 2**20
    assert c5["pairs_exact"] and c5["hist_total_exact"] and c5["pi_within_5_sigma"]


def test_bench_c4_digests_identical_at_1_and_2_ranks():
    """bench.py's C4 row (10^12 numbers, stream space split over the ranks):
    the per-call digest list is the same whether one rank owns every stream
    or two ranks (gloo, sharing the one GPU here) split them."""
    base = [os.path.join(ROOT, "bench.py"), "--steps", "4", "--warmup", "3", "--streams", "65536", "--c4-only",
            "--e2e-steps", "1", "--no-cpu-baseline"]
    r1 = subprocess.run([sys.executable] + base, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r1.returncode == 0, r1.stderr[-3000:]
    d1 = json.loads([ln for ln in r1.stdout.splitlines() if ln.startswith("{")][-1])["secondary"]["c4_sharded_1e12"]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}"] + base + ["--gpus", "2"]
    env = dict(os.environ, CIPRNG_BENCH_BACKEND="gloo")
    r2 = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r2.returncode == 0, r2.stderr[-3000:]
    d2 = json.loads([ln for ln in r2.stdout.splitlines() if ln.startswith("{")][-1])["secondary"]["c4_sharded_1e12"]
    assert d1["n_gpus"] == 1 and d2["n_gpus"] == 2 and d1["numbers"] == d2["numbers"] == 1000727379968
    assert d1["digest_list_sha256"] == d2["digest_list_sha256"]
    assert d1["digests_first3"] == d2["digests_first3"]
