#!/bin/bash
O=gpurun_out/${1:-s31}; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py -q -k "v1_ or v3_ or v34" -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
timeout 300 python tools/exp_oddn.py > $O/oddn.json 2>$O/err.txt
echo done > $O/done
