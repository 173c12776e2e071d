#!/bin/bash
# A/B of library builds: bench lines (DD/TD/QD config-2 shape) for the
# default libmpcore.so and every build/ab/*.so (MPCORE_LIB), interleaved
cd "$GRAFT_REPO_ROOT"; o=gpurun_out/s3/ab; mkdir -p $o
libs="default $(ls build/ab/*.so 2>/dev/null)"
for rep in ${REPS:-1 2}; do
for k in ${KS:-2 3 4}; do
  for L in $libs; do
    if [ "$L" = default ]; then unset MPCORE_LIB; else export MPCORE_LIB=$PWD/$L; fi
    timeout 300 python bench.py --k $k --steps ${STEPS:-10} --warmup 3 --no-cpu --no-e2e --no-extras > $o/b.json 2> $o/b.err || tail -3 $o/b.err
    python -c "
import json; d=json.loads(open('$o/b.json').read().strip().splitlines()[-1])
print('rep $rep k=$k %-28s %.3f ms  upd %.3f step %.3f' % ('$(basename $L)', d['ms_per_step'], d['roofline']['frac'], d['roofline']['whole_step_frac']), {a: round(b, 2) for a, b in d['kernels_ms_per_step'].items()})"
  done
done
done
unset MPCORE_LIB
