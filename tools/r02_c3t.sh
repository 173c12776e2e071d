#!/bin/bash
# config 3: the refinement tests, then the bench line (20 steps) and the
# host phase log of one run
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_convert.py tests/test_gpu_config3.py tests/test_gpu_config3_fullsize.py tests/test_gpu_ffi.py tests/test_gpu_api.py 2>&1 | tail -2
timeout 300 python bench.py --config 3 --steps 20 --warmup 3 --no-cpu > /tmp/c3.json 2>/dev/null
python -c "import json; d=json.load(open('/tmp/c3.json')); print(round(d['value']*1e3,2), 'ms', {a: round(v*1e3,2) for a,v in d['timings_s'].items()})"
MPCORE_REFINE_TIMERS=1 timeout 300 python bench.py --config 3 --steps 1 --warmup 1 --no-cpu 2>&1 >/dev/null | tail -14
