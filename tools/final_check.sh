timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/final/default.json 2> gpurun_out/final/default.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final/ref.json 2> gpurun_out/final/ref.err
timeout 600 python bench.py --config 3 --steps 7 --warmup 2 > gpurun_out/final/c3.json 2> gpurun_out/final/c3.err
for f in default ref c3; do python -c "
import json; d=json.load(open('gpurun_out/final/$f.json')); e=d.get('e2e') or {}; r=d.get('roofline') or {}
print('$f', d['value'], d['unit'], d['ms_per_step'], 'e2e', e.get('value'), 'frac', r.get('frac'), r.get('whole_step_frac'), 'cpu', (d.get('cpu_baseline') or {}).get('value'), d.get('clocks', {}).get('reasons'))"; done
