#!/bin/bash
# one build->measure cycle: full GPU suite, then bench lines for DD/TD/QD
# (config 2 shape), optionally the panel probe.  TAG names the output dir.
cd "$GRAFT_REPO_ROOT"; o=gpurun_out/s3/${TAG:-cyc}; mkdir -p $o
if [ -z "$NOTEST" ]; then
  timeout 900 python -m pytest -m gpu -x -q -p no:cacheprovider tests > $o/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $o/pytest_gpu.log
  tail -3 $o/pytest_gpu.log
fi
for k in ${KS:-2 3 4}; do
  timeout 300 python bench.py --k $k --steps ${STEPS:-10} --warmup 3 --no-cpu > $o/bench_k$k.json 2> $o/bench_k$k.err || tail -5 $o/bench_k$k.err
  python - <<PY
import json
d = json.loads(open("$o/bench_k$k.json").read().strip().splitlines()[-1])
print("k=$k", "%.1f GF/s" % d["value"], "%.3f ms" % d["ms_per_step"], "e2e %.1f" % d["e2e"]["value"],
      {a: round(b, 2) for a, b in d["kernels_ms_per_step"].items()},
      "upd %.3f" % d["roofline"]["frac"], "step %.3f" % d["roofline"]["whole_step_frac"])
PY
done
[ -n "$PROBE" ] && TAG=$TAG bash tools/s3_panelprobe.sh > /dev/null 2>&1 && grep -A3 'stamps\|period (cycles)' gpurun_out/s3/panelprobe$TAG.txt | grep -v '^J\|^ *[0-9]' 
exit 0
