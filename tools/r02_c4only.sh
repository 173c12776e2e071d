#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/r02
timeout 900 python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu --dist-trace gpurun_out/r02/dist_panels_n32768.txt > gpurun_out/r02/c4b.json 2>gpurun_out/r02/c4b.err; echo "c4 rc=$?"
cat gpurun_out/r02/c4b.json | head -c 3000
grep -v "NCCL INFO" gpurun_out/r02/c4b.err | tail -20
ls -la gpurun_out/r02/dist_panels_n32768.txt
