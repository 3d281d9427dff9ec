#!/bin/bash
# V1 store kernel: persistent prefetching grid sweep (CIPRNG_V1_GRID = CTAs per SM, 0 = one tile per warp)
O=gpurun_out/${1:-s10}; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py -q -k "shapes or default_tables" --maxfail=5 -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
for cfg in "2 0" "2 6" "2 5" "2 4" "2 3" "4 0" "4 3" "1 0" "1 12" "1 8" "8 0"; do set -- $cfg
  CIPRNG_V1_COLS=32 CIPRNG_V1_WPB=$1 CIPRNG_V1_GRID=$2 timeout 120 python bench.py --no-cpu-baseline --no-secondary --steps 400 --e2e-steps 1 > $O/b_w$1_g$2.json 2>>$O/err.txt
done
for f in $O/b_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['value'], round(d['roofline']['frac'],4))"; done > $O/summary.txt
CIPRNG_V1_COLS=32 CIPRNG_V1_WPB=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:v1_fast -s 2 -c 1 -o $O/prof_c32 -f python tools/prof_kernels.py v1 4 > $O/ncu1.txt 2>&1
CIPRNG_V1_COLS=32 CIPRNG_V1_WPB=2 CIPRNG_V1_GRID=6 timeout 600 ncu --set full --import-source on --clock-control none -k regex:v1_fast -s 2 -c 1 -o $O/prof_c32_g6 -f python tools/prof_kernels.py v1 4 > $O/ncu2.txt 2>&1
echo done > $O/done
