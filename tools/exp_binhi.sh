#!/bin/bash
# consumer bin index x >> 24: SHF (default) vs IMAD.HI (-DCIPRNG_EXP_BIN_HI); parity under the experiment build
O=gpurun_out/binhi; mkdir -p $O
for rep in 1 2; do
for ex in "" "-DCIPRNG_EXP_BIN_HI"; do
  CIPRNG_NVCC_EXTRA="$ex" python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > $O/build.log 2>&1
  CIPRNG_NVCC_EXTRA="$ex" timeout 300 python tools/exp_consume.py >> $O/res.jsonl 2>> $O/err.txt
  if [ "$ex" != "" ] && [ $rep = 1 ]; then
    timeout 600 python -m pytest tests/test_parity_gpu.py -q -k "consume or c5" -p no:cacheprovider > $O/tests_binhi.log 2>&1; echo rc=$? >> $O/tests_binhi.log
  fi
done
done
python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
echo done > $O/done
