#!/bin/bash
O=gpurun_out/${1:-s14}; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
for e in 0 1; do CIPRNG_EVICT_FIRST=$e timeout 300 python tools/exp_v2.py > $O/v2_e$e.json 2>>$O/err.txt; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:v2_kernel -s 2 -c 1 -o $O/prof_v2 -f python tools/prof_kernels.py v2 4 > $O/ncu.txt 2>&1
echo done > $O/done
