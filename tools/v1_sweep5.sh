#!/bin/bash
O=gpurun_out/${1:-s17}; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
for cfg in "32 3" "32 4" "32 5" "32 6" "32 8"; do set -- $cfg
  for rep in 1 2; do
  CIPRNG_V1_COLS=$1 CIPRNG_V1_WPB=$2 timeout 120 python bench.py --no-cpu-baseline --no-secondary --steps 300 --e2e-steps 1 > $O/b_c$1_w$2_r$rep.json 2>>$O/err.txt
  done
done
for f in $O/b_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['value'], round(d['roofline']['frac'],4), d['steady_state']['value'])"; done > $O/summary.txt
echo done > $O/done
