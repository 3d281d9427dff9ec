#!/bin/bash
# C4 at one GPU (2^23 streams: 192 MiB of state planes, > L2): state L2 prefetch / policy knobs
O=gpurun_out/c4st; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
for cfg in "default" "CIPRNG_V1_PF=1" "CIPRNG_EVICT_FIRST=0" "CIPRNG_V1_PF=1 CIPRNG_V1_WPB=4" "CIPRNG_V1_WPB=1" "CIPRNG_V1_WPB=4" "default"; do
  env $([ "$cfg" = default ] || echo $cfg) timeout 300 python bench.py --c4-only --steps 10 --no-cpu-baseline --e2e-steps 1 2>>$O/err.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['secondary']['c4_sharded_1e12']; print(json.dumps({'cfg':'$cfg','c4':c['value'],'sha':c['digest_list_sha256'][:12]}))" >> $O/res.jsonl
done
echo done > $O/done
