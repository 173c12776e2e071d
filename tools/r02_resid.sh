#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest -q -x tests/test_gpu_long_residual.py tests/test_gpu_config3.py tests/test_gpu_config3_fullsize.py 2>&1 | tail -3
for v in 0 2 3; do
  MPCORE_RESIDUAL_VARIANT=$v timeout 300 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu > /tmp/c3_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/c3_$v.json')); print('variant $v', d['value'], d['timings_s'])"
done
