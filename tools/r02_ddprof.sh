#!/bin/bash
# DD n = 2048 LU + solve: launch list, and one --set full capture of a wide
# trailing-update launch
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/r02/prof
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/r02/prof/launches_dd2048.csv python tools/prof_run.py 2 2048 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r02/prof/launches_dd2048.csv --by-kernel
MPCORE_NO_GRAPH=1 timeout 900 ncu --set full --import-source on --clock-control none \
  -k "regex:gemm_kernel" -s 21 -c 1 -o gpurun_out/r02/prof/dd_update python tools/prof_run.py 2 2048 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r02/prof/dd_update.ncu-rep 15
