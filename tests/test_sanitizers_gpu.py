"""compute-sanitizer over every kernel family (SURVEY s4 layer 6 / s5 race
detection).  tests/sanitize_cases.py runs small shapes of the 2-D TMA, 3-D
band, staged-STG and direct store paths, the consumers, the battery,
generate_host, the digest, Blum-Goldwasser and Algorithm 1 -- each also
checked against the oracle -- and this test runs it under memcheck,
racecheck (shared-memory hazards: the per-warp TMA staging buffers, the
consumer histograms), synccheck and initcheck, requiring zero reports.
The paper's Alg. 4/5 read and write shared cells without synchronisation
(PAPER.md P:971-973); here the exchange is a register shuffle
and shared memory only stages stores and histograms, which racecheck checks.

The pool's compute-sanitizer was closed during round 2 (its wrapper refuses
with exit 86: runs under it had left GPUs needing a reset).  The sanitizer
passes therefore run only with CIPRNG_RUN_SANITIZERS=1 and skip on a
refusal; the clean logs of the round-2 runs are in profiles/r2_sanitizer/.
The cases themselves run without a sanitizer in test_sanitize_cases_plain."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
CASES = ["tma2d", "band3d", "staged", "direct", "jump", "consume", "battery", "host", "digest", "bg", "chaos"]
# initcheck does not see writes made by the async proxy (cp.async.bulk.tensor
# stores): every word a TMA-path kernel wrote is reported as uninitialised
# when it is copied back, although each case checks every word against the
# oracle (gpurun_out/sanitizer_initcheck.log of r2: 94064 reports, all
# "cudaMemcpy source", all on TMA-written buffers).  initcheck therefore
# runs the cases whose stores are ordinary STG.
INITCHECK_CASES = ["staged", "direct", "jump", "consume", "battery", "digest", "bg", "chaos"]


def test_sanitize_cases_plain():
    """The sanitizer cases without a sanitizer: each kernel family on small
    shapes, every result checked against the oracle."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "sanitize_cases.py"), *CASES],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0 and "sanitize cases ok" in r.stdout, (r.stdout + r.stderr)[-3000:]


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_sanitizer_clean(tool):
    if os.environ.get("CIPRNG_RUN_SANITIZERS", "0") != "1":
        pytest.skip("compute-sanitizer runs only with CIPRNG_RUN_SANITIZERS=1 (closed on this pool; "
                    "round-2 clean logs in profiles/r2_sanitizer/)")
    if not os.path.exists(SAN):
        pytest.fail("compute-sanitizer not found")
    extra = []
    if tool == "memcheck":
        extra = ["--leak-check", "no"]
    elif tool == "racecheck":
        extra = ["--racecheck-report", "all"]
    log_dir = os.path.join(ROOT, "gpurun_out")
    os.makedirs(log_dir, exist_ok=True)
    log = os.path.join(log_dir, f"sanitizer_{tool}.log")
    cases = INITCHECK_CASES if tool == "initcheck" else CASES
    cmd = [SAN, "--tool", tool, "--error-exitcode", "97", "--print-limit", "50", *extra,
           "--kernel-name", "kns=ciprng", sys.executable, os.path.join(ROOT, "tests", "sanitize_cases.py"), *cases]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    with open(log, "w") as fh:
        fh.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    tail = (r.stdout + r.stderr)[-3000:]
    if r.returncode == 86 and "closed" in tail:
        pytest.skip(f"{tool}: compute-sanitizer refused by the pool wrapper")
    assert r.returncode == 0, f"{tool}: exit {r.returncode}\n{tail}"
    assert "sanitize cases ok" in r.stdout, tail
    summary = "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" if tool == "racecheck" \
        else "ERROR SUMMARY: 0 errors"
    assert summary in (r.stdout + r.stderr), tail
