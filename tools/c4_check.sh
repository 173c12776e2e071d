for f in "" "--dist-protocol"; do
timeout 600 python bench.py --config 4 --dim 2048 --steps 2 --warmup 1 $f > gpurun_out/c4a.json 2> gpurun_out/c4a.err; tail -2 gpurun_out/c4a.err | grep -v NCCL
python -c "
import json; d=json.load(open('gpurun_out/c4a.json')); print('$f', d['value'], d['ms_per_step'], d['check'], d['config']['parallelism'][:40])"
done
timeout 1200 python bench.py --config 4 --steps 2 --warmup 1 > gpurun_out/c4b.json 2> gpurun_out/c4b.err
python -c "
import json; d=json.load(open('gpurun_out/c4b.json')); print('n=32768', d['value'], d['ms_per_step'], d['check'], d['roofline']['frac'])"
