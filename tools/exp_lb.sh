#!/bin/bash
# explicit minimum of 1 CTA/SM (relaxed register budget) on the V0 / V1 / V3 kernels
O=gpurun_out/lb; mkdir -p $O
for rep in 1 2; do
for ex in "" "-DCIPRNG_EXP_LB_MIN1"; do
  CIPRNG_NVCC_EXTRA="$ex" python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > $O/build.log 2>&1
  CIPRNG_NVCC_EXTRA="$ex" timeout 300 python tools/exp_consume.py >> $O/res.jsonl 2>> $O/err.txt
  CIPRNG_NVCC_EXTRA="$ex" timeout 300 python tools/exp_v3_shape.py >> $O/res.jsonl 2>> $O/err.txt
  CIPRNG_NVCC_EXTRA="$ex" timeout 300 python tools/exp_v0_shape.py >> $O/res.jsonl 2>> $O/err.txt
  timeout 300 python bench.py --no-secondary --no-cpu-baseline --steps 100 --e2e-steps 1 2>>$O/err.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'build':'$ex','v1_store':d['value'],'steady':d['steady_state']['value']}))" >> $O/res.jsonl
done
done
python -c "import sys; sys.path.insert(0,'.'); from paper_1112_5239_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
echo done > $O/done
