O=gpurun_out/mont; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_parity_gpu.py -q -k "modsq or v2_kernel_kinds" -p no:cacheprovider > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
timeout 600 python tools/exp_v2_kinds.py 1 10 > $O/kinds.json 2> $O/kinds.err
CIPRNG_V2_KIND=10 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"v2_kernel" -s 2 -c 1 -o $O/prof_v2mont -f python tools/prof_kernels.py v2 4 > $O/ncu_v2mont.txt 2>&1
echo done > $O/done
