#!/bin/bash
# V1 consumer launch bounds: default (72 regs), (128, 8) = 64 regs, (128) = 80 regs
O=gpurun_out/v1c; mkdir -p $O
for rep in 1 2; do
for ex in "" "-DCIPRNG_EXP_V1C_THREADS=128 -DCIPRNG_EXP_V1C_MINB=8" "-DCIPRNG_EXP_V1C_THREADS=128"; do
  CIPRNG_NVCC_EXTRA="$ex" python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > $O/build.log 2>&1
  CIPRNG_NVCC_EXTRA="$ex" timeout 300 python tools/exp_consume.py >> $O/res.jsonl 2>> $O/err.txt
  if [ "$ex" = "-DCIPRNG_EXP_V1C_THREADS=128 -DCIPRNG_EXP_V1C_MINB=8" ] && [ $rep = 1 ]; then
    timeout 600 python -m pytest tests/test_parity_gpu.py -q -k "consume or c5" -p no:cacheprovider > $O/tests_v1c.log 2>&1; echo rc=$? >> $O/tests_v1c.log
  fi
done
done
python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
echo done > $O/done
