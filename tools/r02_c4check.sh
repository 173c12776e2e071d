#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest -q -x tests/test_gpu_dist_native.py 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 2 > /tmp/c2.json 2>/tmp/c2.err; echo "c2 rc=$?"; python -c "import json; d=json.load(open('/tmp/c2.json')); print(d['check'], d['value'])"
tail -3 /tmp/c2.err
timeout 900 python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu --dist-trace gpurun_out/r02/dist_panels_n32768.txt > /tmp/c4.json 2>/tmp/c4.err; echo "c4 rc=$?"; python -c "import json; d=json.load(open('/tmp/c4.json')); print(d['check'], d['value'], d['phases_ms_rank0'])"
tail -3 /tmp/c4.err
