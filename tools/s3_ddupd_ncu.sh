#!/bin/bash
# ncu --set full of one wide DD trailing-update launch (panel 10 of an
# n = 2048 one-call LU; direct launches)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out/s3/prof
python tools/prof_run.py 2 2048 > gpurun_out/s3/prof/plain.log 2>&1 && \
MPCORE_NO_GRAPH=1 timeout 900 ncu --set full --import-source on --clock-control none \
  -k "regex:gemm_kernel" -s ${SKIP:-21} -c 1 -o gpurun_out/s3/prof/dd_update_rest \
  python tools/prof_run.py 2 2048 > gpurun_out/s3/prof/dd_update.log 2>&1
echo "rc=$?"
