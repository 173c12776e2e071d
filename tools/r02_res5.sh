#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_long_residual.py 2>&1 | tail -2
for cfg in "MPCORE_X=1" "MPCORE_RESIDUAL_VARIANT=2"; do
  env $cfg timeout 300 python bench.py --config 3 --steps 20 --warmup 3 --no-cpu > /tmp/c3.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/c3.json')); print('$cfg', round(d['value']*1e3,2), 'ms', {a: round(v*1e3,2) for a,v in d['timings_s'].items()})"
done
