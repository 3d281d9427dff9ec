#!/bin/bash
# V3 TMA store box width / warps per CTA (ALU-bound kernel: more resident warps?)
O=gpurun_out/v3shape; mkdir -p $O
for rep in 1 2; do
for ex in "" "-DCIPRNG_V3_COLS=16" "-DCIPRNG_V3_COLS=16 -DCIPRNG_V3_WPB=4" "-DCIPRNG_V3_COLS=8 -DCIPRNG_V3_WPB=4" "-DCIPRNG_V3_WPB=1" "-DCIPRNG_V3_COLS=16 -DCIPRNG_V3_WPB=1"; do
  CIPRNG_NVCC_EXTRA="$ex" python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > $O/build.log 2>&1
  CIPRNG_NVCC_EXTRA="$ex" timeout 300 python tools/exp_v3_shape.py >> $O/res.jsonl 2>> $O/err.txt
done
done
python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
echo done > $O/done
