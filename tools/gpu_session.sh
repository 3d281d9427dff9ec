#!/bin/bash
# One gpurun session: tests, bench, ncu.  Usage: bash tools/gpu_session.sh TAG [what...]
TAG=${1:-r1}; shift
WHAT=${@:-"smoke tests bench ncu"}
O=gpurun_out/$TAG; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
for w in $WHAT; do
case $w in
smoke) timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log ;;
tests) timeout 1500 python -m pytest tests -m gpu -q --maxfail=20 --timeout=900 -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log ;;
fasttests) timeout 900 python -m pytest tests -m "gpu and not slow" -q --maxfail=20 --timeout=600 -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log ;;
bench) timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo rc=$? >> $O/bench.err ;;
benchpaths) for sp in 1 2; do timeout 300 python bench.py --store-path $sp --no-cpu-baseline --no-secondary --steps 400 > $O/bench_sp$sp.json 2>> $O/bench.err; done
  CIPRNG_V1_SMEM_STG=1 timeout 300 python bench.py --store-path 1 --no-cpu-baseline --no-secondary --steps 400 > $O/bench_sp1_smemstg.json 2>> $O/bench.err ;;
ref) timeout 300 python bench.py --impl reference --steps 20 --warmup 3 > $O/bench_ref.json 2>> $O/bench.err ;;
ncu)
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_bench_stdout.txt 2>&1
  for k in ${NCU_KINDS:-v1 v1direct v2 v0 v3 v4 consume consume_v0 consume_v2 consume_v3 battery cbg alg1 c1 digest}; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:"v1_fast|v2_kernel|v0_kernel|v1_general|comb_|cbg_|alg1_|v0_jump|digest_" -s 2 -c 1 -o $O/prof_$k -f python tools/prof_kernels.py $k 4 > $O/ncu_$k.txt 2>&1
  done ;;
pipes) timeout 300 python tools/pipe_bench.py > $O/pipes.json 2> $O/pipes.err ;;
esac
done
echo session-done > $O/done
