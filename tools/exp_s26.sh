#!/bin/bash
O=gpurun_out/${1:-s26}; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
echo done > $O/done
