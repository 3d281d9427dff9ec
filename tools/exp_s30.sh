#!/bin/bash
O=gpurun_out/${1:-s30}; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_nccl_gpu.py -q -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
echo done > $O/done
