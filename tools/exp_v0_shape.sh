#!/bin/bash
# V0/V4 store CTA shape: the wave count of the grid (32768 warp tiles at 2^20 streams)
O=gpurun_out/v0shape; mkdir -p $O
for rep in 1 2; do
for ex in "" "-DCIPRNG_V0_WPB=4 -DCIPRNG_V0_PAD_SMEM=28000" "-DCIPRNG_V0_WPB=4 -DCIPRNG_V0_MINB=11" "-DCIPRNG_V0_PAD_SMEM=56000" "-DCIPRNG_V0_WPB=4"; do
  CIPRNG_NVCC_EXTRA="$ex" python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > $O/build.log 2>&1
  grep -A3 "v0_kernelINS_9StoreSinkELb0ELi0" paper_1112_5239_b200/build/gen_v0.cu.ptxas.txt | grep -E "registers|spill" | tr '\n' ' ' >> $O/regs.txt; echo " <- $ex" >> $O/regs.txt
  CIPRNG_NVCC_EXTRA="$ex" timeout 300 python tools/exp_v0_shape.py >> $O/res.jsonl 2>> $O/err.txt
done
done
python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
echo done > $O/done
