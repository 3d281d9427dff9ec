O=gpurun_out/s8; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -q --maxfail=20 --timeout=600 -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
for pdl in 1 0; do
 for cfg in "32 2 0" "64 1 0" "128 1 0" "64 2 -1"; do set -- $cfg
  CIPRNG_PDL=$pdl CIPRNG_V1_COLS=$1 CIPRNG_V1_WPB=$2 CIPRNG_V1_PERSIST=$3 timeout 120 python bench.py --no-cpu-baseline --no-secondary --steps 400 --e2e-steps 1 > $O/b_pdl${pdl}_c$1_w$2_p$3.json 2>>$O/err.txt
 done
done
timeout 300 python bench.py --steps 200 > $O/bench.json 2>>$O/err.txt
echo done > $O/done
