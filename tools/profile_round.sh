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
for spec in "update:regex:gemm_kernel:40" "panel:regex:panel_kernel:20" \
            "swaptrsm:regex:swap_trsm:20" "fwd:regex:sweep_kernel<3, 0>:0" \
            "bwd:regex:sweep_kernel<3, 1>:0"; do
  IFS=: read name kind re skip <<< "$spec"
  MPCORE_NO_GRAPH=1 ncu --set full --import-source on --clock-control none \
    -k "$kind:$re" -s $skip -c 1 -o gpurun_out/prof/td_$name \
    python tools/prof_run.py 3 2048 > gpurun_out/prof/td_$name.log 2>&1
done
ls -la gpurun_out/prof
