"""The a7 row on a real GPU: the sharded consumer (dist.sharded_consume:
prng_consume on each rank's shard, then one SUM all-reduce of the 258 u64
statistics) and the sharded verification digests (dist.sharded_digests),
launched with torchrun one process per rank, compared counter by counter and
digest by digest with the UNSHARDED oracle over the same stream space.

* world size 2 over gloo: both ranks share the one GPU of the test box; the
  collective really runs (asserted through dist.COLLECTIVES_RUN);
* world size 2 over NCCL: needs two GPUs (NCCL cannot put two ranks on one
  device), so it runs only where torch.cuda.device_count() >= 2;
* world size 1 over NCCL: the process-group plumbing only -- at world size 1
  allreduce_sum_ has nothing to exchange and runs no collective (asserted).
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_stats_digests(variant, seed, S, n, calls, digest_calls):
    st = O.init_states(variant, seed, 0, S)
    ref = np.zeros(258, np.uint64)
    for _ in range(calls):
        O.stats(O.generate(variant, st, n), ref)
    st = O.init_states(variant, seed, 0, S)
    digs = [O.digest(O.generate(variant, st, n), 0) for _ in range(digest_calls)]
    return [int(v) for v in ref], digs


@pytest.mark.parametrize("variant", [0, 1, 2, 3])
@pytest.mark.parametrize("backend,nproc", [("gloo", 2), ("nccl", 2), ("nccl", 1)])
def test_torchrun_sharded_consume_matches_oracle(variant, backend, nproc):
    if backend == "nccl" and nproc > torch.cuda.device_count():
        pytest.skip(f"NCCL with {nproc} ranks needs {nproc} GPUs (have {torch.cuda.device_count()})")
    # 96 groups of 32 streams: ranks own 48 groups each; n even (consumer pairs)
    S, n, calls, dcalls = 3072, 64, 2, 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "tools", "dist_consume.py"),
           "--streams", str(S), "--rounds", str(n), "--calls", str(calls), "--variant", str(variant),
           "--backend", backend, "--digest-calls", str(dcalls)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["world_size"] == nproc and d["backend"] == backend
    # one all-reduce for the statistics, one per digest call -- and none at world size 1
    assert d["collectives_run"] == (1 + dcalls if nproc > 1 else 0)
    ref, ref_d = _oracle_stats_digests(variant, d["seed"], S, n, calls, dcalls)
    assert d["stats"] == ref
    assert d["digests"] == ref_d


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


def test_bench_gpus_2_self_launches_without_torchrun():
    """`python bench.py --gpus 2` with no torchrun around it (the way the
    driver may invoke the N-GPU runs) starts two ranks itself; here they share
    the one GPU over gloo.  Exactly one line, n_gpus == 2."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CIPRNG_BENCH_BACKEND"] = "gloo"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "4", "--warmup",
                        "3", "--streams", "65536", "--no-secondary", "--e2e-steps", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["global_streams"] == 2 * 65536


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
    # the fixed-space verification counters equal the oracle-checked ones at 1 rank
    r1 = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "4", "--warmup", "3",
                         "--streams", "65536", "--c5-only", "--e2e-steps", "1", "--no-cpu-baseline"],
                        capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r1.returncode == 0, r1.stderr[-3000:]
    d1 = json.loads([ln for ln in r1.stdout.splitlines() if ln.startswith("{")][-1])
    assert d1["secondary"]["c5_consume_allreduce"]["verify"]["stats_sha256"] == c5["verify"]["stats_sha256"]


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
