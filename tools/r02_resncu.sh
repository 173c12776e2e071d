#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/r02/prof
timeout 900 ncu --set full --import-source on --clock-control none -k regex:long_residual_split -c 1 -o gpurun_out/r02/prof/resid python bench.py --config 3 --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1
echo rc=$?
python tools/ncu_summary.py gpurun_out/r02/prof/resid.ncu-rep 25
