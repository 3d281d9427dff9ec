#!/bin/bash
O=gpurun_out/${1:-s24}; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 -p no:cacheprovider -k "c5_shape or v3_c2 or c2_full or c3_full" > $O/gpu_tests_slow.log 2>&1; echo rc=$? >> $O/gpu_tests_slow.log
echo done > $O/done
