O=gpurun_out/s7; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
for S in 1048576 4194304; do
 for cfg in "32 2 0" "64 1 0"; do set -- $cfg
  CIPRNG_V1_COLS=$1 CIPRNG_V1_WPB=$2 CIPRNG_V1_PERSIST=$3 timeout 120 python bench.py --no-cpu-baseline --no-secondary --steps 100 --e2e-steps 1 --streams $S > $O/b_S${S}_c$1.json 2>>$O/err.txt
 done
done
CIPRNG_V1_COLS=32 CIPRNG_V1_WPB=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:v1_fast -s 2 -c 1 -o $O/prof_c32 -f python tools/prof_kernels.py v1 4 > $O/ncu_c32.txt 2>&1
CIPRNG_V1_COLS=64 CIPRNG_V1_WPB=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:v1_band -s 2 -c 1 -o $O/prof_c64 -f python tools/prof_kernels.py v1 4 > $O/ncu_c64.txt 2>&1
timeout 600 python tools/c4_sharded.py > $O/c4.json 2> $O/c4.err
timeout 300 python -m pytest tests/test_nccl_gpu.py -q -p no:cacheprovider > $O/nccl_tests.log 2>&1
echo done > $O/done
