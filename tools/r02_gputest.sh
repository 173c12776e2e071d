#!/bin/bash
# GPU test suite (optionally a subset: args passed to pytest)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/r02
timeout 1700 python -m pytest -m gpu -x -q -p no:cacheprovider "${@:-tests}" > gpurun_out/r02/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02/pytest_gpu.log
tail -15 gpurun_out/r02/pytest_gpu.log
