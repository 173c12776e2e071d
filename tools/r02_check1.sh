#!/bin/bash
# round-2 validation: GPU test suite + compute-sanitizer runs
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02/pytest_gpu.log
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  timeout 900 $S --tool $tool --print-limit 50 python tools/sanitize_run.py 3:257 2:513 4:130 > gpurun_out/r02/sanitizer_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/r02/sanitizer_$tool.log
done
tail -3 gpurun_out/r02/pytest_gpu.log
tail -2 gpurun_out/r02/sanitizer_*.log
