#!/bin/bash
O=${1:-gpurun_out/sweep2}; mkdir -p $O
run() { CIPRNG_V1_COLS=$1 CIPRNG_V1_WPB=$2 CIPRNG_V1_PERSIST=$3 timeout 120 python bench.py --no-cpu-baseline --no-secondary --steps 400 --e2e-steps 1 $5 > $O/$4.json 2>>$O/err.txt; }
run 32 2 0 c32_w2
for cols in 64 128; do for wpb in 1 2; do for p in 0 -1; do run $cols $wpb $p c${cols}_w${wpb}_p${p}; done; done; done
run 128 1 -1 c128_w1_p-1_n256 "--streams 8388608 --rounds 256"
run 32 2 0 c32_w2_n256 "--streams 8388608 --rounds 256"
python - "$O" <<'PY'
import json, os, sys
d = sys.argv[1]
rows = []
for f in sorted(os.listdir(d)):
    if f.endswith('.json'):
        try:
            j = json.load(open(os.path.join(d, f)))
            rows.append((j['roofline']['frac'], j['value'], j['roofline']['avg_kernel_ms'], f))
        except Exception as e:
            rows.append((0, 0, 0, f + ' ERR'))
for r in sorted(rows, reverse=True):
    print(f"{r[3]:28s} {r[1]:.4e} frac={r[0]:.4f} kern_ms={r[2]:.4f}")
PY
