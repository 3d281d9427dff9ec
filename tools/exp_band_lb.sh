#!/bin/bash
# V1 band kernel (n >= 192) launch-bounds minimum 0 (default) vs 1 (relaxed registers)
O=gpurun_out/bandlb; mkdir -p $O
for rep in 1 2; do
for ex in "" "-DCIPRNG_EXP_BAND_MINB=1"; do
  CIPRNG_NVCC_EXTRA="$ex" python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > $O/build.log 2>&1
  for shape in "1048576 256" "8388608 256" "1048576 1024"; do
    set -- $shape
    timeout 300 python bench.py --streams $1 --rounds $2 --steps 30 --no-secondary --no-cpu-baseline --e2e-steps 1 2>>$O/err.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'build':'$ex','S':$1,'n':$2,'value':d['value'],'steady':d['steady_state']['value']}))" >> $O/res.jsonl
  done
done
done
python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
echo done > $O/done
