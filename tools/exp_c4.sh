#!/bin/bash
# C4 throughput per V1 store-kernel shape (bench --c4-only, 1 GPU)
O=gpurun_out/c4s; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
for cfg in "32 4" "64 1" "64 2" "128 1" "128 2" "32 2" "32 8" "16 4"; do
  set -- $cfg
  CIPRNG_V1_COLS=$1 CIPRNG_V1_WPB=$2 timeout 300 python bench.py --c4-only --steps 10 --no-cpu-baseline --e2e-steps 1 2>>$O/err.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['secondary']['c4_sharded_1e12']; print(json.dumps({'cols':$1,'wpb':$2,'c4':c['value'],'sha':c['digest_list_sha256'][:12],'c2':d['value']}))" >> $O/res.jsonl
done
