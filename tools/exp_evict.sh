#!/bin/bash
# output evict-first hint on/off vs whether the state planes fit L2 (V1 store, L2 flushed bench)
O=gpurun_out/evict; mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1
for rep in 1 2; do
for shape in "1048576 128" "1048576 256" "8388608 128" "8388608 256" "4194304 128"; do
  set -- $shape
  for ef in 1 0; do
    CIPRNG_EVICT_FIRST=$ef timeout 300 python bench.py --streams $1 --rounds $2 --steps 40 --no-secondary --no-cpu-baseline --e2e-steps 1 2>>$O/err.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'S':$1,'n':$2,'ef':$ef,'value':d['value'],'steady':d['steady_state']['value']}))" >> $O/res.jsonl
  done
done
done
echo done > $O/done
