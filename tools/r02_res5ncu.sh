#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/r02
MPCORE_RESIDUAL_VARIANT=5 timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"long_" -c 8 --csv --log-file gpurun_out/r02/res5.csv python bench.py --config 3 --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open("gpurun_out/r02/res5.csv")))
h=rows[0]
for r in rows[1:]:
    if len(r)==len(h):
        d=dict(zip(h,r)); print(d["Kernel Name"][:40], d["Metric Name"], d["Metric Value"])
PY
