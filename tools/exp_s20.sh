#!/bin/bash
O=gpurun_out/${1:-s20}; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py -q -k "consume or battery or v1_default" --maxfail=5 -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
for rep in 1 2; do timeout 300 python bench.py --no-cpu-baseline --steps 100 --e2e-steps 1 > $O/b_r$rep.json 2>>$O/err.txt; done
for f in $O/b_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['value'], {k: round(v['value']/1e9,1) for k,v in d.get('secondary',{}).items()})"; done > $O/summary.txt
echo done > $O/done
