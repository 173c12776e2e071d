timeout 600 python bench.py --config 3 --steps 3 --warmup 1 > gpurun_out/c3.json 2> gpurun_out/c3.err; tail -2 gpurun_out/c3.err
python -c "
import json; d=json.load(open('gpurun_out/c3.json')); print(d['value'], d['timings_s'], d['result']['iterations'], d.get('cpu_baseline'))"
nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread"
