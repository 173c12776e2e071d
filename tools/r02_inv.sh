#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/r02
timeout 1500 python tools/dist_invariance.py 32768 1 8 2>&1 | tee gpurun_out/r02/dist_invariance_n32768.txt | tail -5
