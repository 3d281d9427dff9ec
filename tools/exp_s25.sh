#!/bin/bash
O=gpurun_out/${1:-s25}; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_parity_gpu.py -q -k "graph" -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
timeout 300 python bench.py --no-cpu-baseline --no-secondary --steps 200 --e2e-steps 1 > $O/bench.json 2>$O/err.txt
echo done > $O/done
