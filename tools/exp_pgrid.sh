#!/bin/bash
# consumer grids: 1 wave of resident CTAs (default) vs 2 waves vs one tile per warp
O=gpurun_out/pgrid; mkdir -p $O
for rep in 1 2; do
for ex in ${PGRID_SET:-"" "-DCIPRNG_PGRID_WAVES=2" "-DCIPRNG_PGRID_WAVES=0"}; do
  CIPRNG_NVCC_EXTRA="$ex" python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > $O/build.log 2>&1
  CIPRNG_NVCC_EXTRA="$ex" timeout 300 python tools/exp_consume.py >> $O/res.jsonl 2>> $O/err.txt
  if [ "$ex" = "-DCIPRNG_PGRID_WAVES=0" ] && [ $rep = 1 ]; then
    timeout 600 python -m pytest tests/test_parity_gpu.py -q -k "consume or c5" -p no:cacheprovider > $O/tests_pgrid.log 2>&1; echo rc=$? >> $O/tests_pgrid.log
  fi
done
done
python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
echo done > $O/done
