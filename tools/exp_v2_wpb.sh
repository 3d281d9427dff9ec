#!/bin/bash
# V2 store / consume warps per CTA with the register budget of a plain __launch_bounds__(threads)
O=gpurun_out/v2wpb; mkdir -p $O
for rep in 1 2; do
for ex in "" "-DCIPRNG_V2_WPB=8"; do
  CIPRNG_NVCC_EXTRA="$ex" python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > $O/build.log 2>&1
  echo "== $ex" >> $O/res.txt
  CIPRNG_NVCC_EXTRA="$ex" timeout 600 python tools/exp_v2_kinds.py 1 >> $O/res.txt 2>> $O/err.txt
  CIPRNG_NVCC_EXTRA="$ex" timeout 300 python tools/exp_consume.py >> $O/res.txt 2>> $O/err.txt
done
done
python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
echo done > $O/done
