O=gpurun_out/s4; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
python tools/pattern_bench.py > $O/pattern.json 2>&1
for shape in "1048576 128" "262144 512" "131072 1024" "8388608 256"; do set -- $shape
  for cols in 16 32; do
  CIPRNG_V1_COLS=$cols CIPRNG_V1_WPB=4 timeout 120 python bench.py --no-cpu-baseline --no-secondary --steps 200 --e2e-steps 1 --streams $1 --n $2 > $O/v1_${1}x${2}_c$cols.json 2>>$O/err.txt
  done
done
timeout 300 python bench.py --no-cpu-baseline --steps 50 --e2e-steps 1 > $O/bench_sec.json 2>>$O/err.txt
echo done > $O/done
