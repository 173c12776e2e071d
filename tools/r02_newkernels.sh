#!/bin/bash
# ncu --set full of the round-2 kernels: IR residual (products, chains),
# IR conversion, distributed back substitution
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/r02/prof
cap() {  # name, kernel regex, launches to skip, command...
  local nm=$1 re=$2 sk=$3; shift 3
  timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$re" -s $sk -c 1 \
    -o gpurun_out/r02/prof/$nm "$@" > gpurun_out/r02/prof/$nm.log 2>&1
  echo "$nm rc=$?"
  python tools/ncu_summary.py gpurun_out/r02/prof/$nm.ncu-rep 8 > gpurun_out/r02/prof/$nm.txt 2>&1
}
cap ir_products long_products2 1 python bench.py --config 3 --steps 1 --warmup 0 --no-cpu
cap ir_chains long_chain 1 python bench.py --config 3 --steps 1 --warmup 0 --no-cpu
cap ir_convert convert_kernel 3 python bench.py --config 3 --steps 1 --warmup 0 --no-cpu
cap dist_back_update back_update 2 python tools/dist_invariance.py 4096 4
ls gpurun_out/r02/prof/*.txt
