#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/r02
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"convert_kernel|headsum|long_residual|sweep|panel_kernel|gemm|memcpy" -c 200 --csv --log-file gpurun_out/r02/c3_launches.csv python bench.py --config 3 --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1
echo rc=$?
python tools/launch_summary.py gpurun_out/r02/c3_launches.csv --by-kernel | head -20
