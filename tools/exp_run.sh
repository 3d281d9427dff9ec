#!/bin/bash
# Experiment builds: for each set of extra nvcc defines (one per argument,
# "" = the default build) rebuild libciprng.so and run a timing script,
# appending one JSON line per build.  Restores the default build at the end.
#   tools/exp_run.sh OUT.jsonl SCRIPT.py [SCRIPT ARGS] -- "" "-DCIPRNG_EXP_X" ...
# e.g. tools/exp_run.sh gpurun_out/s50.jsonl tools/exp_consume.py -- "" "-DCIPRNG_EXP_PAIR_ADDCC"
OUT=$1; SCRIPT=$2; shift 2
ARGS=()
while [[ $# -gt 0 && $1 != "--" ]]; do ARGS+=("$1"); shift; done
shift
mkdir -p "$(dirname "$OUT")"
for ex in "$@"; do
  CIPRNG_NVCC_EXTRA="$ex" python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > "$OUT.build.log" 2>&1 || { echo "{\"build\": \"$ex\", \"error\": \"build failed\"}" >> "$OUT"; continue; }
  CIPRNG_NVCC_EXTRA="$ex" timeout 600 python "$SCRIPT" "${ARGS[@]}" >> "$OUT" 2>> "$OUT.err"
done
python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
