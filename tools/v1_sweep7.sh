#!/bin/bash
# V1: 3-D band boxes (whole 256-byte row pieces) with the L2 hints, vs the 2-D default
O=gpurun_out/${1:-s23}; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
for cfg in "32 2 4" "64 1 1" "64 1 2" "64 1 3" "64 2 1" "64 2 2" "128 1 1" "128 1 2"; do set -- $cfg
  CIPRNG_V1_COLS=$1 CIPRNG_V1_BUFS=$2 CIPRNG_V1_WPB=$3 timeout 300 python -m pytest tests/test_parity_gpu.py -q -k "v1_default" -p no:cacheprovider >> $O/gpu_tests.log 2>&1; echo "cols=$1 bufs=$2 wpb=$3 rc=$?" >> $O/gpu_tests.log
  CIPRNG_V1_COLS=$1 CIPRNG_V1_BUFS=$2 CIPRNG_V1_WPB=$3 timeout 120 python bench.py --no-cpu-baseline --no-secondary --steps 300 --e2e-steps 1 > $O/b_c$1_b$2_w$3.json 2>>$O/err.txt
done
for f in $O/b_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['value'], round(d['roofline']['frac'],4), d['steady_state']['value'])"; done > $O/summary.txt
echo done > $O/done
