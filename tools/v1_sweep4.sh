#!/bin/bash
# V1 TMA store: tiles per warp x warps per CTA x box width, L2-flushed bench
O=gpurun_out/${1:-s16}; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py -q -k "shapes or v1_default" --maxfail=5 -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
for cfg in "32 2 1" "32 2 2" "32 2 3" "32 4 1" "32 4 2" "32 1 2" "16 4 1" "16 8 1" "16 4 2" "8 8 1"; do set -- $cfg
  CIPRNG_V1_COLS=$1 CIPRNG_V1_WPB=$2 CIPRNG_V1_TPW=$3 timeout 120 python bench.py --no-cpu-baseline --no-secondary --steps 300 --e2e-steps 1 > $O/b_c$1_w$2_t$3.json 2>>$O/err.txt
done
for f in $O/b_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['value'], round(d['roofline']['frac'],4), d['steady_state']['value'])"; done > $O/summary.txt
echo done > $O/done
