timeout 600 python bench.py > gpurun_out/b2.json 2> gpurun_out/b2.err; tail -2 gpurun_out/b2.err
python -c "
import json; d=json.load(open('gpurun_out/b2.json')); print('cfg2', d['value'], d['ms_per_step'], d['timing'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'], d['roofline']['whole_step_frac'], d['cpu_baseline']['value'])"
timeout 600 python bench.py --config 1 --k 2 --steps 3 --warmup 2 > gpurun_out/b1.json 2> gpurun_out/b1.err; tail -2 gpurun_out/b1.err
python -c "
import json; d=json.load(open('gpurun_out/b1.json')); print('cfg1', d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'])"
timeout 900 python bench.py --config 4 --dim 8192 --steps 2 --warmup 1 > gpurun_out/b4.json 2> gpurun_out/b4.err; tail -2 gpurun_out/b4.err
python -c "
import json; d=json.load(open('gpurun_out/b4.json')); print('cfg4', d['value'], d['ms_per_step'], d['roofline']['frac'])"
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
