#!/bin/bash
# A/B of the state-planes L2 persisting window and evict-first output stores
O=gpurun_out/${1:-s11}; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py -q -k "v1_default or v3_default or shapes or consume" --maxfail=5 -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
for p in 0 1; do for e in 0 1; do
  CIPRNG_L2PERSIST=$p CIPRNG_EVICT_FIRST=$e timeout 120 python bench.py --no-cpu-baseline --no-secondary --steps 400 --e2e-steps 1 > $O/b_p${p}_e${e}.json 2>>$O/err.txt
done; done
for f in $O/b_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['value'], round(d['roofline']['frac'],4))"; done > $O/summary.txt
python -c "
import torch; p=torch.cuda.get_device_properties(0); print('persistingL2CacheMaxSize', getattr(p,'persisting_l2_cache_max_size',None), 'L2', p.L2_cache_size)" >> $O/summary.txt 2>&1
CIPRNG_L2PERSIST=1 CIPRNG_EVICT_FIRST=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:v1_fast -s 2 -c 1 -o $O/prof_p1e1 -f python tools/prof_kernels.py v1 4 > $O/ncu1.txt 2>&1
echo done > $O/done
