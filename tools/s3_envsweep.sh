#!/bin/bash
# bench lines (config-2 shape) for each value of one environment knob:
#   VAR=MPCORE_PANEL_SPEC_COLS VALS="0 400 700" KS="2 3 4" tools/s3_envsweep.sh
cd "$GRAFT_REPO_ROOT"; o=gpurun_out/s3/sweep; mkdir -p $o
for rep in ${REPS:-1 2}; do
for k in ${KS:-2 3 4}; do
  for v in $VALS; do
    env $VAR=$v timeout 300 python bench.py --k $k --steps ${STEPS:-10} --warmup 3 --no-cpu --no-e2e --no-extras > $o/b.json 2> $o/b.err || tail -3 $o/b.err
    python -c "
import json; d=json.loads(open('$o/b.json').read().strip().splitlines()[-1])
print('rep $rep k=$k $VAR=%-8s %.3f ms  upd %.3f step %.3f' % ('$v', d['ms_per_step'], d['roofline']['frac'], d['roofline']['whole_step_frac']), {a: round(b, 2) for a, b in d['kernels_ms_per_step'].items()})"
  done
done
done
