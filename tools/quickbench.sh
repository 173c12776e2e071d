#!/bin/bash
# tests + TD/QD/DD bench summary (run under gpurun)
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for k in ${KS:-3 4 2}; do
  timeout 300 python bench.py --k $k --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_k$k.json 2> gpurun_out/bench_k$k.err || tail -5 gpurun_out/bench_k$k.err
  python - <<PY
import json
d = json.load(open("gpurun_out/bench_k$k.json"))
print(d["metric"].split()[0], "%.1f GF/s" % d["value"], "%.2f ms" % d["ms_per_step"], "e2e %.1f" % d["e2e"]["value"],
      {a: round(b, 2) for a, b in d["kernels_ms_per_step"].items()},
      "upd %.3f" % d["roofline"]["frac"], "step %.3f" % d["roofline"]["whole_step_frac"])
PY
done
