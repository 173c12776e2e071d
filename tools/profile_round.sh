#!/bin/bash
# Round profile capture (run under gpurun, one GPU):
#  1. launch list of the default bench command (kernel durations, cold,
#     serialised: shares, not absolutes)
#  2. one `ncu --set full` capture per hot kernel of the TD LU+solve
set -x
mkdir -p gpurun_out/prof
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/prof/launches_td2048.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/prof/launches.log 2>&1
cap() {  # name, kernel regex, launches to skip
  MPCORE_NO_GRAPH=1 ncu --set full --import-source on --clock-control none \
    -k "regex:$2" -s $3 -c 1 -o gpurun_out/prof/td_$1 \
    python tools/prof_run.py 3 2048 > gpurun_out/prof/td_$1.log 2>&1
}
cap update_rest gemm_kernel 41
cap panel panel_kernel 20
cap swaptrsm swap_trsm 20
cap sweep_back sweep 0
ls -la gpurun_out/prof
