#!/bin/bash
# consumer pair counter: IADD3.X (default) vs IMAD.X (madc, -DCIPRNG_EXP_MADC); parity under the experiment build
O=gpurun_out/madc; mkdir -p $O
for rep in 1 2; do
for ex in "" "-DCIPRNG_EXP_MADC"; do
  CIPRNG_NVCC_EXTRA="$ex" python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > $O/build.log 2>&1
  CIPRNG_NVCC_EXTRA="$ex" timeout 300 python tools/exp_consume.py >> $O/res.jsonl 2>> $O/err.txt
  if [ "$ex" != "" ] && [ $rep = 1 ]; then
    timeout 600 python -m pytest tests/test_parity_gpu.py -q -k "consume or c5" -p no:cacheprovider > $O/tests_madc.log 2>&1; echo rc=$? >> $O/tests_madc.log
  fi
done
done
python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
echo done > $O/done
