"""bench.py's JSON contract on the reference arm (CPU oracle, no GPU): one
JSON line with the driver's keys, a cpu_baseline and an e2e object, and
nothing printed by non-zero ranks."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra=None, args=()):
    env = dict(os.environ, **(env_extra or {}))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                        "--warmup", "3", *args], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr
    return [ln for ln in r.stdout.splitlines() if ln.strip()]


def test_reference_arm_line():
    lines = _run()
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


def test_reference_arm_nonzero_rank_is_silent():
    assert _run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}) == []


def test_reference_arm_same_config_as_ours():
    """The reference arm times the oracle on OUR arm's workload: every step a
    full C2 call (2^20 streams x 128), CPU model named."""
    d = json.loads(_run(args=("--steps", "1"))[0])
    assert d["config"]["same_config_as_ours"] is True
    assert (d["config"]["streams_per_gpu"], d["config"]["n_per_stream"]) == (2**20, 128)
    assert "cpu_model" in d["cpu_baseline"]


def test_gpus_n_without_torchrun_fails_loudly_without_gpus():
    """`bench.py --gpus N` outside torchrun re-launches itself with N NCCL
    ranks -- and refuses (non-zero exit, a message) when this node has fewer
    than N GPUs (here: none)."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.pop("CIPRNG_BENCH_BACKEND", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 2 and "needs 2 GPUs" in r.stderr
    assert not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
