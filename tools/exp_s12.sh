#!/bin/bash
O=gpurun_out/${1:-s12}; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --maxfail=20 --timeout=900 -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
CIPRNG_EVICT_FIRST=0 timeout 300 python bench.py --no-cpu-baseline --steps 200 --e2e-steps 2 > $O/b_e0.json 2>>$O/err.txt
CIPRNG_EVICT_FIRST=1 timeout 300 python bench.py --no-cpu-baseline --steps 200 --e2e-steps 2 > $O/b_e1.json 2>>$O/err.txt
echo done > $O/done
