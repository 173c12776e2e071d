#!/bin/bash
# config-1 GEMM lines for DD/TD/QD (value, dominant-kernel fraction)
cd "$GRAFT_REPO_ROOT"; o=gpurun_out/s3/${TAG:-gemm}; mkdir -p $o
for k in ${KS:-2 3 4}; do
  timeout 300 python bench.py --config 1 --k $k --steps 3 --warmup 2 --no-cpu --no-e2e > $o/c1_k$k.json 2> $o/c1_k$k.err || tail -3 $o/c1_k$k.err
  python -c "
import json; d=json.loads(open('$o/c1_k$k.json').read().strip().splitlines()[-1])
print('gemm k=$k %.1f GF/s %.2f ms frac %.3f' % (d['value'], d['ms_per_step'], d['roofline']['frac']))"
done
