#!/bin/bash
# V1 TMA store: shared-memory boxes per warp x warps per CTA (c32), L2-flushed bench
O=gpurun_out/${1:-s22}; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
for cfg in "1 4" "1 8" "1 2" "2 4" "3 4" "3 2"; do set -- $cfg
  CIPRNG_V1_BUFS=$1 CIPRNG_V1_WPB=$2 timeout 300 python -m pytest tests/test_parity_gpu.py -q -k "v1_default" -p no:cacheprovider >> $O/gpu_tests.log 2>&1; echo "bufs=$1 wpb=$2 rc=$?" >> $O/gpu_tests.log
  CIPRNG_V1_BUFS=$1 CIPRNG_V1_WPB=$2 timeout 120 python bench.py --no-cpu-baseline --no-secondary --steps 300 --e2e-steps 1 > $O/b_b$1_w$2.json 2>>$O/err.txt
done
for f in $O/b_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['value'], round(d['roofline']['frac'],4), d['steady_state']['value'])"; done > $O/summary.txt
echo done > $O/done
