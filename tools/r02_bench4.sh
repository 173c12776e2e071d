#!/bin/bash
# config 4 (native distributed driver, one rank) + A/B vs the one-call LU
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/r02
NCCL_DEBUG=INFO timeout 900 python bench.py --config 4 --steps 2 --warmup 1 > gpurun_out/r02/bench_c4.json 2> gpurun_out/r02/bench_c4.err
echo "c4 rc=$?"
cat gpurun_out/r02/bench_c4.json
grep -v "NCCL INFO" gpurun_out/r02/bench_c4.err | tail -5
timeout 900 python tools/dist_check.py 8192 32768
