O=gpurun_out/s9; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py -q -k "shapes or default_tables" --maxfail=5 -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
for cfg in "32 2 0" "16 4 0" "64 1 0" "128 1 0" "64 2 -1" "64 1 -1" "128 1 -1" "32 4 0" "16 2 0"; do set -- $cfg
  CIPRNG_V1_COLS=$1 CIPRNG_V1_WPB=$2 CIPRNG_V1_PERSIST=$3 timeout 120 python bench.py --no-cpu-baseline --no-secondary --steps 400 --e2e-steps 1 > $O/b_c$1_w$2_p$3.json 2>>$O/err.txt
done
CIPRNG_V1_COLS=64 CIPRNG_V1_WPB=1 CIPRNG_V1_PERSIST=-1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:v1_band -s 2 -c 1 -o $O/prof_band_persist -f python tools/prof_kernels.py v1 4 > $O/ncu1.txt 2>&1
CIPRNG_V1_COLS=32 CIPRNG_V1_WPB=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:v1_fast -s 2 -c 1 -o $O/prof_c32 -f python tools/prof_kernels.py v1 4 > $O/ncu2.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:v0_kernel -s 2 -c 1 -o $O/prof_v0 -f python tools/prof_kernels.py v0 4 > $O/ncu3.txt 2>&1
echo done > $O/done
