#!/bin/bash
# V1 store-kernel shape sweep (TMA box width x warps/CTA x grid cap).
O=${1:-gpurun_out/sweep}; mkdir -p $O
for cols in 8 16 32; do for wpb in 2 4 8; do for grid in 0 6; do
  CIPRNG_V1_COLS=$cols CIPRNG_V1_WPB=$wpb CIPRNG_V1_GRID=$grid timeout 120 python bench.py --no-cpu-baseline --no-secondary --steps 400 --e2e-steps 1 > $O/c${cols}_w${wpb}_g${grid}.json 2>>$O/err.txt
done; done; done
python - "$O" <<'PY'
import json, os, sys
d = sys.argv[1]
rows = []
for f in sorted(os.listdir(d)):
    if f.endswith('.json'):
        try:
            j = json.load(open(os.path.join(d, f)))
            rows.append((j['roofline']['frac'], j['value'], f))
        except Exception as e:
            rows.append((0, 0, f + ' ERR'))
for r in sorted(rows, reverse=True):
    print(f"{r[2]:24s} {r[1]:.4e} frac={r[0]:.4f}")
PY
