#!/bin/bash
# full GPU suite (verbose log kept) + guard-zone log for profiles/
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/r02
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02/pytest_gpu_full.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02/pytest_gpu_full.log
tail -3 gpurun_out/r02/pytest_gpu_full.log
timeout 600 python -m pytest tests/test_gpu_guards.py -v -p no:cacheprovider > gpurun_out/r02/guards_pytest.log 2>&1
tail -3 gpurun_out/r02/guards_pytest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
