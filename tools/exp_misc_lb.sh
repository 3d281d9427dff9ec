#!/bin/bash
# launch-bounds minimum 0 vs 1 on the chaotic-BG, Alg. 1 and general-table kernels (bench secondary rows)
O=gpurun_out/misclb; mkdir -p $O
for rep in 1 2; do
for ex in "" "-DCIPRNG_EXP_MISC_MINB=1"; do
  CIPRNG_NVCC_EXTRA="$ex" python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > $O/build.log 2>&1
  timeout 600 python bench.py --no-cpu-baseline --steps 20 --e2e-steps 1 2>>$O/err.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['secondary']; print(json.dumps({'build':'$ex','cbg':s['cbg_encrypt']['value'],'alg1':s['alg1_negation_b8']['value'],'v1':d['value']}))" >> $O/res.jsonl
done
done
python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
echo done > $O/done
