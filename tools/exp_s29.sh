#!/bin/bash
O=gpurun_out/${1:-s29}; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
timeout 300 python tools/exp_oddn.py > $O/oddn.json 2>$O/err.txt
timeout 300 python bench.py --no-cpu-baseline --steps 100 --e2e-steps 1 > $O/bench.json 2>>$O/err.txt
timeout 300 python bench.py --store-path 1 --no-cpu-baseline --no-secondary --steps 100 --e2e-steps 1 > $O/bench_direct.json 2>>$O/err.txt
timeout 600 ncu --set full --clock-control none -k regex:"v1_fast" -s 2 -c 1 -o $O/prof_v1direct -f python tools/prof_kernels.py v1direct 4 > $O/ncu.txt 2>&1
echo done > $O/done
