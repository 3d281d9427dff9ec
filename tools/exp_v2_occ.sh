#!/bin/bash
# V2 occupancy / CTA-shape builds (CIPRNG_V2_MINB, CIPRNG_V2_WPB): C3 timing per kind, L2 flushed
O=gpurun_out/v2occ; mkdir -p $O
for ex in "" "-DCIPRNG_V2_MINB=5" "-DCIPRNG_V2_WPB=4" "-DCIPRNG_V2_WPB=4 -DCIPRNG_V2_MINB=10" "-DCIPRNG_V2_MINB=6"; do
  CIPRNG_NVCC_EXTRA="$ex" python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > $O/build.log 2>&1
  echo "== $ex" >> $O/res.txt
  grep -A2 "v2_kernelINS_9StoreSinkELj0ELb1" paper_1112_5239_b200/build/gen_v2.cu.ptxas.txt | tail -2 >> $O/res.txt
  timeout 600 python tools/exp_v2_kinds.py 1 4 >> $O/res.txt 2>> $O/err.txt
done
python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
echo done > $O/done
