#!/bin/bash
# next-panel update on the main stream once the trailing block is narrower
# than MPCORE_NEXT_MAIN_COLS columns (TD/QD); whole-LU time per setting
for k in ${KS:-3 4}; do
  for c in ${COLS:-0 400 700 1000 1300}; do
    MPCORE_NEXT_MAIN_COLS=$c timeout 300 python bench.py --k $k --steps 5 --warmup 3 --no-cpu > gpurun_out/nc.json 2> gpurun_out/nc.err || tail -3 gpurun_out/nc.err
    python -c "
import json; d = json.load(open('gpurun_out/nc.json'))
print('k=$k cols=$c', '%.1f GF/s' % d['value'], '%.2f ms' % d['ms_per_step'], {a: round(b, 2) for a, b in d['kernels_ms_per_step'].items()})"
  done
done
