#!/bin/bash
# consumer experiment builds: default, no histogram, conflict-free bins
O=gpurun_out/cons; mkdir -p $O
for ex in "" "-DCIPRNG_EXP_NOHIST" "-DCIPRNG_EXP_HIST_LANE"; do
  CIPRNG_NVCC_EXTRA="$ex" python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > $O/build.log 2>&1
  CIPRNG_NVCC_EXTRA="$ex" timeout 300 python tools/exp_consume.py >> $O/res.jsonl 2>> $O/err.txt
done
python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
