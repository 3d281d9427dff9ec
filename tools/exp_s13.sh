#!/bin/bash
O=gpurun_out/${1:-s13}; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py -q -k "v1_default or shapes" --maxfail=5 -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
for e in 0 1; do for s in 0 1; do
  CIPRNG_EVICT_FIRST=$e CIPRNG_STATE_EVICT_LAST=$s timeout 300 python bench.py --no-cpu-baseline --no-secondary --steps 300 --e2e-steps 1 > $O/b_e${e}_s${s}.json 2>>$O/err.txt
done; done
for f in $O/b_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['value'], round(d['roofline']['frac'],4), d['steady_state']['value'])"; done > $O/summary.txt
echo done > $O/done
