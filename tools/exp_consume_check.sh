#!/bin/bash
# consumer experiment builds with a parity check: for each define set, rebuild,
# run the V1/V3 consume parity tests, then time the consumers (exp_consume.py)
OUT=$1; shift
mkdir -p "$(dirname "$OUT")"
for ex in "$@"; do
  CIPRNG_NVCC_EXTRA="$ex" python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > "$OUT.build.log" 2>&1 || { echo "{\"build\": \"$ex\", \"error\": \"build failed\"}" >> "$OUT"; continue; }
  r=$(timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_nccl_gpu.py -q -x -k "consume or stats" -p no:cacheprovider 2>&1 | tail -1)
  echo "{\"build\": \"$ex\", \"parity\": \"$r\"}" >> "$OUT"
  CIPRNG_NVCC_EXTRA="$ex" timeout 600 python tools/exp_consume.py >> "$OUT" 2>> "$OUT.err"
done
python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
