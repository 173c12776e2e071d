#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 300 python -m pytest -q -x tests/test_gpu_long_residual.py 2>&1 | tail -1
for np in 1 2 3; do
  MPCORE_RESIDUAL_PRODUCERS=$np timeout 300 python bench.py --config 3 --steps 20 --warmup 3 --no-cpu > /tmp/c3.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/c3.json')); print('producers $np', round(d['value']*1e3,2), 'ms', {a: round(v*1e3,2) for a,v in d['timings_s'].items()})"
done
