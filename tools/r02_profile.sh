#!/bin/bash
# round-2 evidence: full GPU suite, default bench line, ncu launch list of
# the default bench command, one ncu --set full of the wide update (+ the
# per-opcode FP64 counts) and of the back substitution
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/r02/prof
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02/pytest_gpu.log
tail -3 gpurun_out/r02/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02/bench_c2.json 2> gpurun_out/r02/bench_c2.err
echo "bench rc=$?"
cat gpurun_out/r02/bench_c2.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/r02/prof/launches_td2048.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/r02/prof/launches.log 2>&1
echo "launch list rc=$?"
OPS=smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum
cap() {  # name, kernel regex, launches to skip
  MPCORE_NO_GRAPH=1 timeout 900 ncu --set full --metrics $OPS --import-source on --clock-control none \
    -k "regex:$2" -s $3 -c 1 -o gpurun_out/r02/prof/td_$1 \
    python tools/prof_run.py 3 2048 > gpurun_out/r02/prof/td_$1.log 2>&1
  echo "cap $1 rc=$?"
}
cap update_rest gemm_kernel 41
cap sweep_back sweep 0
ls -la gpurun_out/r02/prof
