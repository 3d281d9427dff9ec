#!/bin/bash
# V1 store: 2-D 32-round boxes (wpb 4) vs 3-D band boxes (cols 64, wpb 2) per n, 2^20 streams, L2 flushed
O=gpurun_out/bandn; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
for n in 128 192 256 384 512 1024; do
  for cfg in "32 4" "64 2" "128 1"; do
    set -- $cfg
    CIPRNG_V1_COLS=$1 CIPRNG_V1_WPB=$2 timeout 300 python bench.py --rounds $n --steps 60 --no-secondary --no-cpu-baseline --e2e-steps 1 2>>$O/err.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'n':$n,'cols':$1,'wpb':$2,'value':d['value'],'frac':d['roofline']['frac'],'steady':d['steady_state']['value']}))" >> $O/res.jsonl
  done
done
