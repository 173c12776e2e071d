#!/bin/bash
# every BASELINE config's bench line (and its reference arm) on one B200
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/r02/all
run() { # name, args...
  local nm=$1; shift
  timeout 900 python bench.py "$@" > gpurun_out/r02/all/$nm.json 2> gpurun_out/r02/all/$nm.err
  echo "$nm rc=$?"
}
run c2_td --steps 20 --warmup 5
run c2_qd --k 4 --steps 10 --warmup 3
run c2_dd --k 2 --steps 20 --warmup 5 --no-cpu
run c1_dd --config 1 --k 2 --steps 10 --warmup 3
run c1_td --config 1 --k 3 --steps 5 --warmup 2
run c1_qd --config 1 --k 4 --steps 5 --warmup 2
run c3 --config 3 --steps 10 --warmup 3
run ref_c1 --impl reference --config 1 --steps 1 --warmup 0
run ref_c3 --impl reference --config 3 --steps 1 --warmup 0
run ref_c2 --impl reference --steps 1 --warmup 0
for f in gpurun_out/r02/all/*.json; do echo "== $f"; python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
print(d.get('metric'), round(d.get('value',0),4), d.get('unit'), 'ms', round(d.get('ms_per_step',0),3), 'e2e', (d.get('e2e') or {}).get('value'), 'frac', (d.get('roofline') or {}).get('frac'), 'whole', (d.get('roofline') or {}).get('whole_step_frac'))
"; done
