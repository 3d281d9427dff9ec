#!/bin/bash
O=gpurun_out/${1:-s18}; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py -q -k "v1_ or v2_ or v3_ or shapes or tiles" --maxfail=5 -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
for pf in 0 1; do for rep in 1 2; do
  CIPRNG_V1_PF=$pf timeout 300 python bench.py --no-cpu-baseline --steps 300 --e2e-steps 1 > $O/b_pf${pf}_r$rep.json 2>>$O/err.txt
done; done
for f in $O/b_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['value'], round(d['roofline']['frac'],4), d['steady_state']['value'], {k: round(v['value']/1e9,1) for k,v in d.get('secondary',{}).items()})"; done > $O/summary.txt
echo done > $O/done
