#!/bin/bash
# SURVEY s7 three-way store-path comparison: (a) direct STG, (b) smem transpose + coalesced STG, (c) TMA
O=gpurun_out/${1:-s27}; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_parity_gpu.py -q -k "smem_stg or v1_default" -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
bash tools/gpu_session.sh $(basename $O) benchpaths
for k in v1 v1direct v1smem; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"v1_fast" -s 2 -c 1 -o $O/prof_$k -f python tools/prof_kernels.py $k 4 > $O/ncu_$k.txt 2>&1
done
for f in $O/bench_sp*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['value'], round(d['roofline']['frac'],4), d['config']['store_path'])"; done > $O/summary.txt
echo done > $O/done
