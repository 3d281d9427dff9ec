#!/bin/bash
# V1 C2 store: warps per CTA x boxes per warp, re-swept with the relaxed register budget (88 registers)
O=gpurun_out/v1shape; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
for rep in 1 2; do
for cfg in "4 2" "2 2" "8 2" "4 3" "2 3" "4 1" "8 1"; do
  set -- $cfg
  CIPRNG_V1_COLS=32 CIPRNG_V1_WPB=$1 CIPRNG_V1_BUFS=$2 timeout 300 python bench.py --no-secondary --no-cpu-baseline --steps 100 --e2e-steps 1 2>>$O/err.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'wpb':$1,'bufs':$2,'value':d['value'],'steady':d['steady_state']['value']}))" >> $O/res.jsonl
done
done
echo done > $O/done
